# what makes the 70B-shape (group 8) attention slower than the 8B shape: vary one factor at a time
python -m paper_2506_15155_b200.build
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 10"
run() { n=$1; shift; timeout 600 $B "$@" > gpurun_out/p_$n.log 2>&1; echo "$n: $* -> $(grep -o '"achieved": [0-9.]*' gpurun_out/p_$n.log) $(grep -o '"launch_ms": [0-9.]*' gpurun_out/p_$n.log)"; }
run A --workload c2 --context 8192 --batch 64
run B --workload c2 --layers 80
run C --workload c4 --layers 32
run C2 --workload c4 --layers 32 --tokens-per-chunk 16
run D1 --workload c4 --batch 32 --context 16384
ELLM_ATTN_DYN_DIV=16 run E16 --workload c4
ELLM_ATTN_DYN_DIV=8 run E8 --workload c4
run S2 --workload c4 --emulate-shard 2
run S4 --workload c4 --emulate-shard 4
run S8 --workload c4 --emulate-shard 8
run Z2 --workload c2 --emulate-shard 2
run Z8 --workload c2 --emulate-shard 8
