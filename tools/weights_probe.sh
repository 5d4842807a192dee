python -m paper_2506_15155_b200.build > /dev/null 2>&1
for cfg in "c2 1 1" "c2 1 0" "c4 1 1"; do timeout 900 python tools/attn_weights_probe.py $cfg 2>&1 | tail -6; done
