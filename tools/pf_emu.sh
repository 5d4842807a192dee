python -m paper_2506_15155_b200.build > /dev/null 2>&1
for e in 0 1 2 3; do echo "EMU=$e"; ELLM_PF_EMU=$e timeout 300 python tools/prefill_bench.py 2>&1 | tail -5; done
