#!/bin/bash
# final validation of HEAD on a 4-GPU box: GPU suite, smoke, bench at 1 / 2 / 4 GPUs
O=gpurun_out/r02_final_all
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
CUDA_VISIBLE_DEVICES=0 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
CUDA_VISIBLE_DEVICES=0 python bench.py > $O/bench_1gpu.json 2> $O/bench_1gpu.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_2gpu.json 2> $O/bench_2gpu.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 4 --steps 3 --warmup 3 > $O/bench_4gpu.json 2> $O/bench_4gpu.err
