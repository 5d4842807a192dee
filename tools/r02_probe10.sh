python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
for v in "" d16u1 d8u2 d16u2 d4u4; do
  if [ -n "$v" ]; then export ELLM_LIB_PATH=$PWD/paper_2506_15155_b200/libellm_$v.so; else unset ELLM_LIB_PATH; fi
  echo "== variant ${v:-d8u1}"
  for cfg in "c4 8 p2p 0" "c2 1 none 0"; do timeout 600 python tools/attn_timeline.py $cfg 2>&1 | grep -E "shard|merge_us|end_max|stream_end_max|span"; done
done | tee gpurun_out/timeline10.log
