python -m paper_2506_15155_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py tests/test_gpu_configs.py tests/test_gpu_bench_sequence.py -m gpu -q -x 2>&1 | tail -1
for cfg in "c4 1 none 0" "c2 1 none 0" "c4 8 p2p 0"; do timeout 600 python tools/attn_timeline.py $cfg 2>&1 | grep -E "shard|span|stream_end|merge_us"; done
for w in c2 c4; do timeout 900 python bench.py --workload $w --no-swap --no-cpu-baseline --no-e2e > gpurun_out/mc_$w.log 2>&1; tail -1 gpurun_out/mc_$w.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w', d['value'], d['ms_per_step'], r['achieved'], r['launch_ms'])"; done
