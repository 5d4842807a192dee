python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
for cfg in "c4 8 p2p 0 0" "c4 8 p2p 0 1" "c4 8 p2p 1 1" "c2 1 none 0 0" "c2 1 none 0 1" "c2 1 none 1 1"; do timeout 600 python tools/attn_timeline.py $cfg 2>&1 | grep -E "shard|span|stream_end|merge_us|gap_next|per-SM"; done | tee gpurun_out/timeline15.log
