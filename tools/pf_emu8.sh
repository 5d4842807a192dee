python -m paper_2506_15155_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do for e in 0 1 2 3; do echo -n "EMU=$e/8 pairs: "; ELLM_PF_EMU=$e timeout 300 python tools/prefill_bench.py 2>&1 | tail -5 | awk '{print $(NF-1)}' | tr '\n' ' '; echo; done; done
