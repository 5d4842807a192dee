python -m paper_2506_15155_b200.build > /dev/null 2>&1
echo "== full"; timeout 300 python tools/prefill_bench.py 2>&1 | tail -5
echo "== no MMA (timing only)"; ELLM_LIB_PATH=$PWD/paper_2506_15155_b200/libellm_nomma.so timeout 300 python tools/prefill_bench.py 2>&1 | tail -5
