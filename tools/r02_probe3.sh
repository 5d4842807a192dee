python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_rotation.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/t3.log 2>&1; tail -2 gpurun_out/t3.log
timeout 600 python tools/migrate_probe.py > gpurun_out/migrate_probe.log 2>&1; tail -1 gpurun_out/migrate_probe.log
for g in p2p nccl; do for n in 8 4; do timeout 900 python bench.py --workload c4 --emulate-shard $n --gather $g --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4s${n}_$g.log 2>&1; tail -1 gpurun_out/c4s${n}_$g.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$n $g', d['value'], d['ms_per_step'], r['achieved'], r['launch_ms'], d['gpu_launches'])"; done; done
