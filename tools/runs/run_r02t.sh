#!/bin/bash
O=gpurun_out/r02t
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or poisoned or edge_cases or random or schedules' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 default env:GREM_NO_PREFETCH=1 env:GREM_NO_PDL=1 paper_2502_17846_b200/alt/libgrem_r01.so
GREM_DEBUG_MEM=1 python tools/gpu_time.py friendster 256 5 > $O/friendster256.txt 2> $O/friendster256.err
python tools/gpu_time.py friendster 16 4 >> $O/friendster256.txt 2>&1
