python -m paper_2506_15155_b200.build > gpurun_out/build.log 2>&1
for e in 0 2 3 4; do echo "EMU=$e"; ELLM_PF_EMU=$e timeout 300 python tools/prefill_bench.py 2>&1 | tail -5; done > gpurun_out/pf_emu.log; cat gpurun_out/pf_emu.log
timeout 600 python -m pytest tests/test_gpu_prefill.py -m gpu -q -x 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:paged_attn -s 40 -c 2 -o gpurun_out/c4s8_full python bench.py --workload c4 --emulate-shard 8 --steps 1 --warmup 1 --profile --no-swap --no-cpu-baseline --no-e2e > gpurun_out/c4s8_ncu.log 2>&1; tail -2 gpurun_out/c4s8_ncu.log
cat > /tmp/pf_one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from tools.prefill_bench import run
torch.cuda.profiler.start()
run(2, 32768, 4096, iters=1)
torch.cuda.profiler.stop()
PY
PF_L=32 timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill -s 2 -c 1 -o gpurun_out/pf_full python /tmp/pf_one.py > gpurun_out/pf_ncu.log 2>&1; tail -2 gpurun_out/pf_ncu.log
