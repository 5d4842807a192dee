python -m paper_2506_15155_b200.build > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/f8_tests.log 2>&1; tail -2 gpurun_out/f8_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f8_smoke.log 2>&1; tail -1 gpurun_out/f8_smoke.log
timeout 1200 python bench.py > gpurun_out/f8_c2.log 2>&1; tail -1 gpurun_out/f8_c2.log | cut -c1-200
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f8_ref.log 2>&1; tail -1 gpurun_out/f8_ref.log | cut -c1-150
