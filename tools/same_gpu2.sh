# The N>1 bench path (fused gather, folded waits, max-over-ranks timing) with 2 ranks sharing one GPU
# (CUDA IPC windows, gloo process group): a functional check, not a scaling number.
python -m paper_2506_15155_b200.build > /dev/null 2>&1
ELLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --batch 8 --no-swap --no-cpu-baseline > gpurun_out/same_gpu2.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/same_gpu2.log | cut -c1-600
