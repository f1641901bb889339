#!/bin/bash
O=gpurun_out/r02m
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or poisoned or edge_cases or random or schedules or variants or hooks or store' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
GREM_DEBUG_MEM=1 python tools/gpu_time.py papers100m 16 6 > $O/memdbg.txt 2>&1
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 paper_2502_17846_b200/alt/libgrem_r01.so default env:GREM_NO_DEVICE_LOOP=1
SUBTREE_PROFILE=0 python tools/gpu_subtree.py 1 > $O/subtree1.txt 2>&1
GREM_NO_DEVICE_LOOP=1 SUBTREE_PROFILE=0 python tools/gpu_subtree.py 1 > $O/subtree1_nodl.txt 2>&1
