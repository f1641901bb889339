#!/bin/bash
# k_split_edges tile size (256 / 512 / 1024 threads x 8 edges)
O=gpurun_out/r02aw
mkdir -p $O
A=paper_2502_17846_b200/alt
GREM_LIB=$PWD/$A/libgrem_split1024.so python -m pytest tests -m gpu -x -q -k 'golden or schedules or extract or split' > $O/pytest1024.log 2>&1; echo "rc=$?" >> $O/pytest1024.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default $A/libgrem_split512.so $A/libgrem_split1024.so
for v in default $A/libgrem_split512.so $A/libgrem_split1024.so; do
  if [ $v = default ]; then python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1
  else GREM_LIB=$PWD/$v python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1; fi
done
