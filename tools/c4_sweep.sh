# C4 (group 8) vs C2 (group 4) attention GB/s across tokens-per-chunk; then the C5 lockstep test and bench
set -x
python -m paper_2506_15155_b200.build
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 10"
for T in 16 32 64; do timeout 600 $B --workload c4 --tokens-per-chunk $T > gpurun_out/c4_T$T.log 2>&1; grep -o '"roofline": {[^}]*}' gpurun_out/c4_T$T.log; done
for T in 16 32; do timeout 600 $B --workload c2 --tokens-per-chunk $T > gpurun_out/c2_T$T.log 2>&1; grep -o '"roofline": {[^}]*}' gpurun_out/c2_T$T.log; done
timeout 600 $B --workload c4 --batch 32 > gpurun_out/c4_b32.log 2>&1; grep -o '"roofline": {[^}]*}' gpurun_out/c4_b32.log
timeout 900 python -m pytest tests/test_gpu_c5_serve.py -q -x > gpurun_out/c5_test.log 2>&1; tail -30 gpurun_out/c5_test.log
timeout 900 python bench.py --workload c5 > gpurun_out/bench_c5.log 2>&1; tail -30 gpurun_out/bench_c5.log | cut -c1-4000
