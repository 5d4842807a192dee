python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_rotation.py -m gpu -q -x > gpurun_out/t4.log 2>&1; tail -2 gpurun_out/t4.log
timeout 300 python tools/prefill_bench.py > gpurun_out/pf4.log 2>&1; cat gpurun_out/pf4.log | tail -5
for sc in gpu sys; do ELLM_GATHER_SCOPE=$sc timeout 900 python bench.py --workload c4 --emulate-shard 8 --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4s8_$sc.log 2>&1; tail -1 gpurun_out/c4s8_$sc.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('8 $sc', d['value'], d['ms_per_step'], r['achieved'], r['launch_ms'], d['gpu_launches'])"; done
bash tools/sanitize.sh
