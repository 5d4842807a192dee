python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_parity.py tests/test_gpu_c5_serve.py tests/test_gpu_prefill.py -m gpu -q -x > gpurun_out/t5.log 2>&1; tail -2 gpurun_out/t5.log
(cd tools && timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool racecheck ./racecheck_mbarrier_probe > ../gpurun_out/san_probe_racecheck.log 2>&1; tail -3 ../gpurun_out/san_probe_racecheck.log)
for sc in sys gpu; do ELLM_GATHER_SCOPE=$sc timeout 900 python bench.py --workload c4 --emulate-shard 8 --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4s8_$sc.log 2>&1; tail -1 gpurun_out/c4s8_$sc.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('8 $sc', d['value'], d['ms_per_step'], r['achieved'], r['launch_ms'], d['gpu_launches'])"; done
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | cut -c1-300
