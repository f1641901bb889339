#!/bin/bash
O=gpurun_out/r02z
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or schedules' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
GREM_DEBUG_MEM=1 python tools/gpu_time.py friendster 256 10 > $O/f256.txt 2> $O/f256.err
echo "rc=$?" >> $O/f256.txt
python tools/gpu_time.py papers100m 16 10 > $O/papers.txt 2>&1
GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_r01.so python tools/gpu_time.py papers100m 16 10 >> $O/papers.txt 2>&1
