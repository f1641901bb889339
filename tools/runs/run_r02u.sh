#!/bin/bash
O=gpurun_out/r02u
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or schedules or random or hooks' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
python tools/gpu_time.py papers100m 16 12 > $O/papers.txt 2>&1
GREM_DEBUG_MEM=1 python tools/gpu_time.py friendster 256 6 > $O/friendster256.txt 2> $O/friendster256.err
python tools/gpu_time.py papers100m 16 12 >> $O/papers.txt 2>&1
GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_r01.so python tools/gpu_time.py papers100m 16 12 >> $O/papers.txt 2>&1
