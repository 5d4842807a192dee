python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
for cfg in "c4 8 p2p 0" "c2 1 none 0" "c4 1 none 0"; do timeout 600 python tools/attn_timeline.py $cfg 2>&1 | tail -16; done | tee gpurun_out/timeline13.log
