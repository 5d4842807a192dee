python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
for cfg in "c4 8 p2p 0" "c2 1 none 0"; do ELLM_ATTN_RANGE_ROT=1 timeout 600 python tools/attn_timeline.py $cfg 2>&1 | tail -16; done | tee gpurun_out/timeline14.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
