python -m paper_2506_15155_b200.build > /dev/null 2>&1
for cfg in "c4 8" "c4 4" "c2 1" "c4 1"; do timeout 900 python tools/ramp_probe.py $cfg 2>&1 | tail -6; done
