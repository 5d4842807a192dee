python -m paper_2506_15155_b200.build > /dev/null
timeout 300 tools/slab_read 150 short > gpurun_out/slabg.log 2>&1; cat gpurun_out/slabg.log
echo "--- prefill L=32 rotated"; PF_L=32 timeout 300 python tools/prefill_bench.py
echo "--- prefill L=32 canonical"; ELLM_ROTATE=0 PF_L=32 timeout 300 python tools/prefill_bench.py
