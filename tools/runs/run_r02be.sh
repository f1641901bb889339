#!/bin/bash
# compact tiles of 2^13 nodes (2 CTAs/SM, twice the record re-reads) vs 2^14
O=gpurun_out/r02be
mkdir -p $O
GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_sub13.so python -m pytest tests -m gpu -x -q -k 'golden or schedules or random' > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default paper_2502_17846_b200/alt/libgrem_sub13.so
PHASE_K=1 python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1
PHASE_K=1 GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_sub13.so python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1
