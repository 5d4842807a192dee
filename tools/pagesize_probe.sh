# H2D-vs-decode interference as a function of pool size and read footprint (tools/overlap_probe.py)
python -m paper_2506_15155_b200.build >/dev/null
for cfg in "32 16" "32 8" "24 24" "16 16" "32 32"; do echo "== batch/decoding $cfg"; timeout 400 python tools/overlap_probe.py $cfg > gpurun_out/ov_b.log 2>&1; grep -v "^{\|thp" gpurun_out/ov_b.log | cut -c1-120; done
