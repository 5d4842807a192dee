# ncu --set full of the C4 (70B shape, group 8) attention launch
python -m paper_2506_15155_b200.build
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:paged_attn -c 1 \
  -o gpurun_out/attn_c4_full python bench.py --workload c4 --steps 1 --warmup 1 --profile --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4_ncu.log 2>&1
tail -3 gpurun_out/c4_ncu.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:paged_attn -c 1 \
  -o gpurun_out/attn_c4_T64_full python bench.py --workload c4 --tokens-per-chunk 64 --steps 1 --warmup 1 --profile --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4_ncu64.log 2>&1
tail -3 gpurun_out/c4_ncu64.log | cut -c1-300
