#!/bin/bash
O=gpurun_out/r02aa
mkdir -p $O
python bench.py --no-cpu > $O/bench.json 2> $O/bench.err
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 paper_2502_17846_b200/alt/libgrem_r01.so default
python tools/gpu_time.py friendster 256 8 > $O/f256.txt 2>&1
python bench.py --no-cpu > $O/bench2.json 2> $O/bench2.err
