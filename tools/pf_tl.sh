python -m paper_2506_15155_b200.build > /dev/null 2>&1
echo "== full"; timeout 300 python tools/pf_timeline.py
echo "== no MMA"; ELLM_LIB_PATH=$PWD/paper_2506_15155_b200/libellm_nomma.so timeout 300 python tools/pf_timeline.py
