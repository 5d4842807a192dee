# C3 value and e2e vs the copy-engine piece cap (ELLM_CE_MAX_COPY: swap copies split into pieces
# of at most this many bytes, so a step's small input / output copies on the same engines do not
# queue behind one large swap copy). usage: bash tools/c3_capsweep.sh "0 33554432 8388608"
python -m paper_2506_15155_b200.build > /dev/null 2>&1
for cap in ${1:-0 33554432 8388608}; do
  ELLM_CE_MAX_COPY=$cap timeout 1500 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/c3cap_$cap.log 2>&1
  tail -1 gpurun_out/c3cap_$cap.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['c3']; print('cap $cap', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], c['swap_overhead_frac'], json.dumps(c['decode_ms_per_step_by_swap_phase']), c['swap_out_ms'], c['swap_in_ms'])" || tail -3 gpurun_out/c3cap_$cap.log
done
