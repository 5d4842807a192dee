# f4 timing experiments: the prefill kernel with parts removed (results are wrong; timing only)
python -m paper_2506_15155_b200.build > /dev/null 2>&1
for v in "" 1 2 3; do
  if [ -n "$v" ]; then export ELLM_LIB_PATH=$PWD/paper_2506_15155_b200/libellm_pfdbg$v.so; else unset ELLM_LIB_PATH; fi
  echo "== variant ${v:-full}"; timeout 300 python tools/prefill_bench.py 2>&1 | tail -5
done
