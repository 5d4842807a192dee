python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
for cfg in "c4 8 p2p 0 0" "c4 8 p2p 0 1" "c4 8 p2p 1 0"; do timeout 600 python tools/attn_timeline.py $cfg 2>&1 | grep -E "shard|stream_end|per-SM|mapping|blockIdx"; done | tee gpurun_out/timeline16.log
