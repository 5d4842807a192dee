python -m paper_2506_15155_b200.build > /dev/null
cat > /tmp/pf_one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from tools.prefill_bench import run
torch.cuda.profiler.start()
run(2, 32768, 4096, iters=1)
torch.cuda.profiler.stop()
PY
PF_L=32 timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill -s 2 -c 1 -o gpurun_out/pf_full python /tmp/pf_one.py > gpurun_out/pf_ncu.log 2>&1
tail -3 gpurun_out/pf_ncu.log
