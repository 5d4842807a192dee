python -m paper_2506_15155_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_rotation.py tests/test_gpu_prefill_fullsize.py -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/prefill_bench.py 2>&1 | tail -5
timeout 300 python tools/pf_timeline.py 2>&1 | tail -10
