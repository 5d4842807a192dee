python -m paper_2506_15155_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_pdl.py tests/test_gpu_parity.py -q -x > gpurun_out/pdl2_tests.log 2>&1; tail -3 gpurun_out/pdl2_tests.log
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 20"
run() { n=$1; shift; timeout 600 $B "$@" > gpurun_out/p3_$n.log 2>&1; echo "$n: $* -> $(grep -o '"achieved": [0-9.]*' gpurun_out/p3_$n.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/p3_$n.log | head -1) $(tail -1 gpurun_out/p3_$n.log | cut -c1-60)"; }
run c2pdl --workload c2
ELLM_PDL=0 run c2nopdl --workload c2
run c4pdl --workload c4
ELLM_PDL=0 run c4nopdl --workload c4
run c4s8pdl --workload c4 --emulate-shard 8
ELLM_PDL=0 run c4s8nopdl --workload c4 --emulate-shard 8
run c4s4pdl --workload c4 --emulate-shard 4
ELLM_PDL=0 run c4s4nopdl --workload c4 --emulate-shard 4
