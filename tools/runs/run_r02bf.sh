#!/bin/bash
# occupancy knobs of the delta count / round-down kernels re-checked on the final build
O=gpurun_out/r02bf
mkdir -p $O
A=paper_2502_17846_b200/alt
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default $A/libgrem_cd3.so $A/libgrem_rd3.so
