python -m paper_2506_15155_b200.build > /dev/null
for e in 2 4; do ELLM_PF_EMU=$e timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x 2>&1 | tail -1; done
for e in 0 2 4; do echo "--- EMU=$e"; ELLM_PF_EMU=$e timeout 300 python tools/prefill_bench.py; done
