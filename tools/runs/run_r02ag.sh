#!/bin/bash
# unrolled k_cut_packed / k_row_counts_bits vs the committed build
O=gpurun_out/r02ag
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or schedules or seed or cut' > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default paper_2502_17846_b200/alt/libgrem_head.so
python tools/phase_ab.py papers100m 16 > $O/phases.txt 2>&1
GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_head.so python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1
