# GPU tests, then the emulated N-way shard step (real N>1 call sequence, folded gather waits).
python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for n in 2 4 8; do timeout 900 python bench.py --workload c4 --emulate-shard $n --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4s$n.log 2>&1; tail -1 gpurun_out/c4s$n.log | cut -c1-200; done
for n in 2 4 8; do ELLM_PDL=0 timeout 900 python bench.py --workload c4 --emulate-shard $n --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4s${n}_nopdl.log 2>&1; tail -1 gpurun_out/c4s${n}_nopdl.log | cut -c1-200; done
