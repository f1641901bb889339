#!/bin/bash
O=gpurun_out/r02ac
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or schedules or random' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 default env:GREM_GREEN_SPARSE_SMS=0 env:GREM_GREEN_SPARSE_SMS=16 env:GREM_GREEN_SPARSE_SMS=48
GREM_DEBUG_LEVELS=1 python tools/gpu_levels.py papers100m 16 > $O/timeline.txt 2>&1
