python -m paper_2506_15155_b200.build > /dev/null 2>&1
(cd tools && ./tmem_bw) > gpurun_out/tmem_bw.log 2>&1; cat gpurun_out/tmem_bw.log
for cfg in "ce 0" "ce 67108864" "ce 8388608" "staged 0" "sm 0" "mixed 0"; do set -- $cfg
  ELLM_CE_MAX_COPY=$2 timeout 900 python bench.py --workload c3 --swap-mode $1 --no-cpu-baseline --no-e2e > gpurun_out/c3_$1_$2.log 2>&1
  tail -1 gpurun_out/c3_$1_$2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['c3']; print('$1 $2', d['value'], d['ms_per_step'], c['isolated_decode_ms_per_step'], c['swap_overhead_frac'], c['swap_round_ms'])"
done
