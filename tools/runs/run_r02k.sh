#!/bin/bash
O=gpurun_out/r02k
mkdir -p $O
for v in paper_2502_17846_b200/alt/libgrem_r01.so default paper_2502_17846_b200/alt/libgrem_r01.so default; do
    if [ $v = default ]; then python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1;
    else GREM_LIB=$PWD/$v python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1; fi
done
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 default paper_2502_17846_b200/alt/libgrem_sc512.so env:GREM_FINAL_CUT_PASS=1
