python -m paper_2506_15155_b200.build > /dev/null
echo "--- prefill L=32 rotated (groups of 8)"; PF_L=32 timeout 300 python tools/prefill_bench.py
echo "--- prefill L=32 canonical"; ELLM_ROTATE=0 PF_L=32 timeout 300 python tools/prefill_bench.py
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rot2_tests.log 2>&1; tail -3 gpurun_out/rot2_tests.log
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 10"
run() { n=$1; shift; timeout 600 $B "$@" > gpurun_out/r2_$n.log 2>&1; echo "$n: $* -> $(grep -o '"achieved": [0-9.]*' gpurun_out/r2_$n.log) $(grep -o '"f4_prefill": {[^}]*}' gpurun_out/r2_$n.log | grep -o '"tflops": [0-9.]*') $(tail -1 gpurun_out/r2_$n.log | cut -c1-60)"; }
run c4rot --workload c4
run c2rot --workload c2
run c4s2 --workload c4 --emulate-shard 2
run c4s4 --workload c4 --emulate-shard 4
run c4s8 --workload c4 --emulate-shard 8
