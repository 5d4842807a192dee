python -m paper_2506_15155_b200.build > /dev/null
timeout 1200 python bench.py --workload c4 > gpurun_out/f3_c4.log 2>&1; tail -1 gpurun_out/f3_c4.log | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:paged_attn -c 3 \
  -o gpurun_out/f3_c4s8_full python bench.py --workload c4 --emulate-shard 8 --steps 1 --warmup 1 --profile --no-swap --no-cpu-baseline --no-e2e > gpurun_out/f3_c4s8_ncu.log 2>&1
tail -2 gpurun_out/f3_c4s8_ncu.log | cut -c1-200
