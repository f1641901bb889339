#!/bin/bash
O=gpurun_out/r02au
mkdir -p $O
for r in 1 2 3; do
  python tools/e2e_time.py papers100m 16 6 >> $O/e2e.txt 2>&1
  GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_head.so python tools/e2e_time.py papers100m 16 6 >> $O/e2e.txt 2>&1
done
