python -m paper_2506_15155_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pdl.py tests/test_gpu_configs.py -q -x > gpurun_out/fv_tests.log 2>&1; tail -2 gpurun_out/fv_tests.log
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 20"
run() { n=$1; shift; timeout 600 $B "$@" > gpurun_out/fv_$n.log 2>&1; echo "$n: $* -> $(grep -o '"achieved": [0-9.]*' gpurun_out/fv_$n.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/fv_$n.log | head -1) $(tail -1 gpurun_out/fv_$n.log | cut -c1-50)"; }
run c4s8 --workload c4 --emulate-shard 8
run c2s8 --workload c2 --emulate-shard 8
run c4s4 --workload c4 --emulate-shard 4
run c2 --workload c2
