python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_rotation.py -m gpu -q -x 2>&1 | tail -1
for e in 0 2; do echo "EMU=$e"; ELLM_PF_EMU=$e timeout 300 python tools/prefill_bench.py 2>&1 | tail -5; done > gpurun_out/pf_emu7.log; cat gpurun_out/pf_emu7.log
