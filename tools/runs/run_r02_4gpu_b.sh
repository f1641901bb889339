#!/bin/bash
# sharded host upload (1/W per rank + NCCL all-gather): e2e at 2 and 4 GPUs
O=gpurun_out/r02_4gpu_b
mkdir -p $O
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_2gpu.json 2> $O/bench_2gpu.err
echo "rc=$?" >> $O/bench_2gpu.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 4 --steps 3 --warmup 3 > $O/bench_4gpu.json 2> $O/bench_4gpu.err
echo "rc=$?" >> $O/bench_4gpu.err
