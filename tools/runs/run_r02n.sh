#!/bin/bash
# 2-GPU: sharded bench (torchrun) + shard tests
O=gpurun_out/r02n
mkdir -p $O
nvidia-smi -L > $O/smi.txt
python -m pytest tests/test_shard.py -m gpu -q > $O/pytest_shard.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_2gpu.json 2> $O/bench_2gpu.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $O/bench_2gpu_ref.json 2> $O/bench_2gpu_ref.err
