set -x
timeout 900 python -m pytest tests/test_gpu_gather.py -q -x -s > gpurun_out/gather_tests.log 2>&1; tail -30 gpurun_out/gather_tests.log
ELLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --batch 8 --steps 10 --warmup 3 --no-swap --no-cpu-baseline > gpurun_out/bench_same_gpu2.log 2>&1; tail -c 2500 gpurun_out/bench_same_gpu2.log
