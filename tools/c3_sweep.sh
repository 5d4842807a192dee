# C3 policy sweep: resident-set size x swap engine (bench.py --workload c3)
python -m paper_2506_15155_b200.build >/dev/null
for a in "--resident 9 --swap-mode mixed" "--resident 9 --swap-mode sm" "--resident 6 --swap-mode mixed" "--resident 9 --swap-mode mixed --swap-every 96"; do
  echo "== $a"; timeout 900 python bench.py --workload c3 --no-cpu-baseline --no-e2e $a > gpurun_out/c3_sweep.log 2>&1
  tail -1 gpurun_out/c3_sweep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['c3']['isolated_decode_ms_per_step'], d['c3']['swap_overhead_frac'], d['c3']['swap_gbs_bidir_serial'], d['roofline']['achieved'])" || tail -5 gpurun_out/c3_sweep.log
done
