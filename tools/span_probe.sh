# attention GB/s vs pool VA span (layers per chunk) at fixed per-launch bytes
python -m paper_2506_15155_b200.build
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 10"
run() { n=$1; shift; timeout 600 $B "$@" > gpurun_out/s_$n.log 2>&1; echo "$n: $* -> $(grep -o '"achieved": [0-9.]*' gpurun_out/s_$n.log) $(grep -o '"mapped_gib": [0-9.]*' gpurun_out/s_$n.log) $(tail -1 gpurun_out/s_$n.log | cut -c1-80)"; }
for L in 40 48 56 64 72; do run c4L$L --workload c4 --layers $L; done
run c2L40 --workload c2 --layers 40
run c2L36 --workload c2 --layers 36
