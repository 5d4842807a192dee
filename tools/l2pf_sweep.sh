# L2 prefetch depth before the PDL / folded-gather wait (ELLM_ATTN_L2PF), same box, interleaved:
# emulated 8- and 4-way C4 shards and C2 at N = 1. usage: bash tools/l2pf_sweep.sh "0 4 8" [reps]
python -m paper_2506_15155_b200.build > /dev/null 2>&1
vals=${1:-"0 4 8"}; reps=${2:-2}
for rep in $(seq $reps); do
for cfg in "c4 8" "c4 4" "c2 0"; do set -- $cfg; w=$1; n=$2
for pf in $vals; do
  extra=""; [ "$n" != "0" ] && extra="--emulate-shard $n"
  ELLM_ATTN_L2PF=$pf timeout 600 python bench.py --workload $w $extra --steps 20 --no-swap --no-cpu-baseline --no-e2e > gpurun_out/l2pf_${w}_${n}_${pf}_$rep.log 2>&1
  tail -1 gpurun_out/l2pf_${w}_${n}_${pf}_$rep.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w x$n pf=$pf rep=$rep', d['value'], r['achieved'], r['launch_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/l2pf_${w}_${n}_${pf}_$rep.log
done; done; done
