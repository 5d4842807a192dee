# HEAD verification on one B200: GPU tests, smoke, default bench, c4 bench, reference arm
set -x
python -m paper_2506_15155_b200.build
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_tests_full.log 2>&1; tail -25 gpurun_out/gpu_tests_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | head -c 3000
timeout 1200 python bench.py --workload c4 --no-swap > gpurun_out/bench_c4.log 2>&1; tail -3 gpurun_out/bench_c4.log | head -c 3000
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | head -c 1500
