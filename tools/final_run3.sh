# end-of-round HEAD verification: GPU tests, smoke, default bench, C4 / C5 lines, reference arm
python -m paper_2506_15155_b200.build > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/f4_tests.log 2>&1; tail -9 gpurun_out/f4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; tail -1 gpurun_out/f4_smoke.log
timeout 1200 python bench.py > gpurun_out/f4_c2.log 2>&1; tail -1 gpurun_out/f4_c2.log | cut -c1-400
timeout 1200 python bench.py --workload c4 > gpurun_out/f4_c4.log 2>&1; tail -1 gpurun_out/f4_c4.log | cut -c1-400
timeout 900 python bench.py --workload c5 > gpurun_out/f4_c5.log 2>&1; tail -1 gpurun_out/f4_c5.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f4_ref.log 2>&1; tail -1 gpurun_out/f4_ref.log | cut -c1-200
