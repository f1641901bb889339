#!/bin/bash
O=gpurun_out/r02at
mkdir -p $O
python bench.py > $O/bench1.json 2> $O/bench1.err
python bench.py > $O/bench2.json 2> $O/bench2.err
GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_head.so python bench.py > $O/bench_head.json 2> $O/bench_head.err
python bench.py --steps 6 > $O/bench3.json 2> $O/bench3.err
