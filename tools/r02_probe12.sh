python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
for dv in 0 8 16 32; do echo "== DYN_DIV $dv"; ELLM_ATTN_DYN_DIV=$dv timeout 600 python tools/attn_timeline.py c4 8 p2p 0 2>&1 | grep -E "span|stream_end|merge_us|gap_next|first_data"; done | tee gpurun_out/timeline12.log
