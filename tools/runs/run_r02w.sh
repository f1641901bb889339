#!/bin/bash
O=gpurun_out/r02w
mkdir -p $O
GREM_DEBUG_MEM=1 python tools/gpu_time.py friendster 256 8 > $O/friendster256.txt 2> $O/friendster256.err
python -m pytest tests/test_gpu_sweep.py -s -q > $O/sweep.log 2>&1
python tools/gpu_time.py friendster 64 5 >> $O/friendster256.txt 2>&1
python tools/gpu_time.py friendster 4 4 >> $O/friendster256.txt 2>&1
