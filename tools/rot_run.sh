# rotated-slab layout: full GPU tests, then C4 / C2 / C5 with and without rotation
python -m paper_2506_15155_b200.build
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rot_tests.log 2>&1; tail -15 gpurun_out/rot_tests.log
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 10"
run() { n=$1; shift; timeout 600 $B "$@" > gpurun_out/r_$n.log 2>&1; echo "$n: $* -> $(grep -o '"achieved": [0-9.]*' gpurun_out/r_$n.log) $(grep -o '"f4_prefill": {[^}]*}' gpurun_out/r_$n.log | grep -o '"tflops": [0-9.]*') $(tail -1 gpurun_out/r_$n.log | cut -c1-60)"; }
run c4rot --workload c4
ELLM_ROTATE=0 run c4canon --workload c4
run c2rot --workload c2
ELLM_ROTATE=0 run c2canon --workload c2
run c4s2 --workload c4 --emulate-shard 2
run c4s8 --workload c4 --emulate-shard 8
run c2s8 --workload c2 --emulate-shard 8
