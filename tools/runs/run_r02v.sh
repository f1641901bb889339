#!/bin/bash
O=gpurun_out/r02v
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or schedules' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
GREM_DEBUG_MEM=1 python tools/gpu_time.py friendster 256 8 > $O/friendster256.txt 2> $O/friendster256.err
python tools/gpu_time.py papers100m 16 12 > $O/papers.txt 2>&1
SUBTREE_PROFILE=0 python tools/gpu_subtree.py 1 > $O/subtree1.txt 2>&1
