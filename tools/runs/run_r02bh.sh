#!/bin/bash
# k_count_delta with 8 edges in flight per thread (3 or 4 CTAs/SM) vs 4
O=gpurun_out/r02bh
mkdir -p $O
A=paper_2502_17846_b200/alt
GREM_LIB=$PWD/$A/libgrem_du8.so python -m pytest tests -m gpu -x -q -k 'golden or schedules' > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default $A/libgrem_du8.so $A/libgrem_du8m4.so
