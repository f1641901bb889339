#!/bin/bash
O=gpurun_out/r02p2
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or random' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 default env:GREM_NO_STAGED_DELTA=1 paper_2502_17846_b200/alt/libgrem_cd3.so
python tools/gpu_time.py friendster 16 4 > $O/friendster.txt 2>&1
python tools/gpu_time.py friendster 256 4 >> $O/friendster.txt 2>&1
python tools/gpu_time.py products 16 6 >> $O/friendster.txt 2>&1
