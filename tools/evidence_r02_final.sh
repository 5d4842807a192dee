# Round-2 final evidence at HEAD on one B200 (outputs gpurun_out/f_*). Part A: GPU tests, smoke,
# default bench (C2), reference arm, ncu launch list of the timed C2 steps + one full capture of
# the C2 attention launch. Part B: C3 / C4 / C5 lines, emulated 2/4/8-way shards, sanitizer.
# usage: bash tools/evidence_r02_final.sh A|B
set -x
python -m paper_2506_15155_b200.build > /dev/null
if [ "$1" = "A" ]; then
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/f_tests.log 2>&1; tail -20 gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
timeout 1200 python bench.py > gpurun_out/f_c2.log 2>&1; tail -1 gpurun_out/f_c2.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref.log 2>&1; tail -1 gpurun_out/f_ref.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 1 --profile --no-swap --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:paged_attn -c 1 \
  -o gpurun_out/f_c2_full python bench.py --steps 1 --warmup 1 --profile --no-swap --no-cpu-baseline --no-e2e > gpurun_out/f_c2_ncu.log 2>&1
fi
if [ "$1" = "B" ]; then
timeout 1500 python bench.py --workload c3 > gpurun_out/f_c3.log 2>&1; tail -1 gpurun_out/f_c3.log | cut -c1-300
timeout 1200 python bench.py --workload c4 > gpurun_out/f_c4.log 2>&1; tail -1 gpurun_out/f_c4.log | cut -c1-300
for n in 2 4 8; do timeout 900 python bench.py --workload c4 --emulate-shard $n --no-swap --no-cpu-baseline > gpurun_out/f_c4s$n.log 2>&1; tail -1 gpurun_out/f_c4s$n.log | cut -c1-200; done
for n in 2 4 8; do timeout 900 python bench.py --workload c2 --emulate-shard $n --no-swap --no-cpu-baseline > gpurun_out/f_c2s$n.log 2>&1; tail -1 gpurun_out/f_c2s$n.log | cut -c1-200; done
timeout 900 python bench.py --workload c5 > gpurun_out/f_c5.log 2>&1; tail -1 gpurun_out/f_c5.log | cut -c1-300
bash tools/sanitize.sh
fi
ls gpurun_out
