python -m paper_2506_15155_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_pdl.py tests/test_gpu_abi.py tests/test_abi.py -q 2>&1 | tail -1
timeout 600 python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/pc_c2.log 2>&1; echo "c2 $(grep -o '"achieved": [0-9.]*' gpurun_out/pc_c2.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/pc_c2.log | head -1)"
timeout 600 python bench.py --workload c5 --no-e2e --no-cpu-baseline > gpurun_out/pc_c5.log 2>&1; echo "c5 $(grep -o '"value": [0-9.]*' gpurun_out/pc_c5.log | head -1) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/pc_c5.log | head -1)"
