#!/bin/bash
# k_bin_hist with the hub prefilter vs HEAD
O=gpurun_out/r02bb
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or schedules or random or hub' > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default paper_2502_17846_b200/alt/libgrem_head.so
python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1
GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_head.so python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1
