#!/bin/bash
# scatter: hub-probe prefilter + odd carry stride, each alone and together, vs HEAD
O=gpurun_out/r02aq
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or schedules or random or hub' > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
A=paper_2502_17846_b200/alt
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default $A/libgrem_bloom.so $A/libgrem_stride.so $A/libgrem_head.so
for v in default $A/libgrem_bloom.so $A/libgrem_stride.so $A/libgrem_head.so; do
  if [ $v = default ]; then PHASE_K=1 python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1
  else PHASE_K=1 GREM_LIB=$PWD/$v python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1; fi
done
