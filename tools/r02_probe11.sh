python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py tests/test_gpu_pdl.py tests/test_gpu_configs.py tests/test_gpu_rotation.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/t11.log 2>&1; tail -2 gpurun_out/t11.log
for cfg in "c4 8 p2p 0" "c4 8 p2p 1" "c4 4 p2p 0" "c2 1 none 0"; do timeout 600 python tools/attn_timeline.py $cfg 2>&1 | tail -13; done | tee gpurun_out/timeline11.log
for n in 8 4 2; do timeout 900 python bench.py --workload c4 --emulate-shard $n --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4s${n}_11.log 2>&1; tail -1 gpurun_out/c4s${n}_11.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$n', d['value'], d['ms_per_step'], r['achieved'], r['launch_ms'], d['gpu_launches'])"; done
