python -m paper_2506_15155_b200.build > /dev/null
timeout 1500 python bench.py --workload c3 > gpurun_out/f10_c3.log 2>&1; tail -1 gpurun_out/f10_c3.log | cut -c1-150
for n in 2 4 8; do timeout 900 python bench.py --workload c4 --emulate-shard $n --no-swap --no-cpu-baseline > gpurun_out/f10_c4s$n.log 2>&1; tail -1 gpurun_out/f10_c4s$n.log | cut -c1-120; done
for n in 2 4 8; do timeout 900 python bench.py --workload c2 --emulate-shard $n --no-swap --no-cpu-baseline > gpurun_out/f10_c2s$n.log 2>&1; tail -1 gpurun_out/f10_c2s$n.log | cut -c1-120; done
