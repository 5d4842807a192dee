# Dynamic tail (ELLM_ATTN_DYN_DIV / _UNIT; dynamic tickets turn PDL off) vs the static split with
# PDL on / off at the emulated 8-way C4 shard. usage: bash tools/dyn_sweep.sh
python -m paper_2506_15155_b200.build > /dev/null 2>&1
run() {  # label, env...
  lab=$1; shift
  env "$@" timeout 600 python bench.py --workload c4 --emulate-shard ${N:-8} --steps 20 --no-swap --no-cpu-baseline --no-e2e > gpurun_out/dyn_$lab.log 2>&1
  tail -1 gpurun_out/dyn_$lab.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lab', d['value'], r['achieved'], r['launch_ms'])" || tail -3 gpurun_out/dyn_$lab.log
}
run static_pdl ELLM_PDL=1
run static_nopdl ELLM_PDL=0
for div in 2 4 8; do for u in 4 8 16; do run div${div}_u$u ELLM_ATTN_DYN_DIV=$div ELLM_ATTN_DYN_UNIT=$u; done; done
