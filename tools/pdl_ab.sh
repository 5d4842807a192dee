python -m paper_2506_15155_b200.build > /dev/null 2>&1
for w in c2 c4; do for pdl in 1 0; do ELLM_PDL=$pdl timeout 900 python bench.py --workload $w --no-swap --no-cpu-baseline --no-e2e > gpurun_out/pdl_${w}_$pdl.log 2>&1; tail -1 gpurun_out/pdl_${w}_$pdl.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w pdl=$pdl', d['value'], d['ms_per_step'], r['achieved'], r['launch_ms'], d['clocks']['sm_mhz'])"; done; done
for n in 8 4; do for pdl in 1 0; do ELLM_PDL=$pdl timeout 900 python bench.py --workload c4 --emulate-shard $n --no-swap --no-cpu-baseline --no-e2e > gpurun_out/pdl_s${n}_$pdl.log 2>&1; tail -1 gpurun_out/pdl_s${n}_$pdl.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4 x$n pdl=$pdl', d['value'], d['ms_per_step'], r['achieved'], r['launch_ms'])"; done; done
