# round-1 evidence at HEAD: GPU tests, prefill A/B, bench lines (C2 default, C4, C5), ncu launch list + C4 full capture
set -x
python -m paper_2506_15155_b200.build > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/final_tests.log 2>&1; tail -14 gpurun_out/final_tests.log
echo "--- prefill L=32 rotated"; PF_L=32 timeout 300 python tools/prefill_bench.py
echo "--- prefill L=32 canonical"; ELLM_ROTATE=0 PF_L=32 timeout 300 python tools/prefill_bench.py
timeout 1200 python bench.py > gpurun_out/final_c2.log 2>&1; tail -1 gpurun_out/final_c2.log | cut -c1-1500
timeout 1200 python bench.py --workload c4 > gpurun_out/final_c4.log 2>&1; tail -1 gpurun_out/final_c4.log | cut -c1-1500
timeout 900 python bench.py --workload c5 > gpurun_out/final_c5.log 2>&1; tail -1 gpurun_out/final_c5.log | cut -c1-800
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --profile --no-swap --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:paged_attn -c 1 \
  -o gpurun_out/final_c4_full python bench.py --workload c4 --steps 1 --warmup 1 --profile --no-swap --no-cpu-baseline --no-e2e > gpurun_out/final_c4_ncu.log 2>&1
ls -la gpurun_out/
