python -m paper_2506_15155_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py -m gpu -q -x 2>&1 | tail -1
for e in 0 1 2; do echo "EMU=$e"; ELLM_PF_EMU=$e timeout 300 python tools/prefill_bench.py 2>&1 | tail -5; done
ELLM_PF_EMU=0 timeout 300 python tools/pf_timeline.py 2>&1 | tail -14
ELLM_PF_EMU=1 timeout 300 python tools/pf_timeline.py 2>&1 | tail -14
