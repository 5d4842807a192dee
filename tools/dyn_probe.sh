python -m paper_2506_15155_b200.build > /dev/null
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 20"
run() { n=$1; shift; timeout 600 $B "$@" > gpurun_out/d_$n.log 2>&1; echo "$n: $* -> $(grep -o '"achieved": [0-9.]*' gpurun_out/d_$n.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/d_$n.log | head -1) $(tail -1 gpurun_out/d_$n.log | cut -c1-50)"; }
for dv in 0 4 8 16; do ELLM_ATTN_DYN_DIV=$dv run c4s8_$dv --workload c4 --emulate-shard 8; done
for dv in 0 4 16; do ELLM_ATTN_DYN_DIV=$dv run c2s8_$dv --workload c2 --emulate-shard 8; done
for dv in 0 16; do ELLM_ATTN_DYN_DIV=$dv run c4_$dv --workload c4; done
timeout 1200 python bench.py --workload c4 > gpurun_out/f3_c4.log 2>&1; tail -1 gpurun_out/f3_c4.log | cut -c1-300
