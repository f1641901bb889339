#!/bin/bash
O=gpurun_out/r02_4gpu
mkdir -p $O
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 3 --warmup 3 > $O/bench_4gpu.json 2> $O/bench_4gpu.err
echo "rc=$?" >> $O/bench_4gpu.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > $O/bench_4gpu_ref.json 2> $O/bench_4gpu_ref.err
echo "rc=$?" >> $O/bench_4gpu_ref.err
