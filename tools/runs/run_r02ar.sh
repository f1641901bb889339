#!/bin/bash
# (1) 4-node composite steps in k_bundle_sim vs the per-node chain; (2) scatter shared-memory footprint variants
O=gpurun_out/r02ar
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or schedules or random or bundle' > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
A=paper_2502_17846_b200/alt
for r in 1 2; do
  python tools/sparse_side.py 4 >> $O/sparse.txt 2>&1
  GREM_LIB=$PWD/$A/libgrem_noblk4.so python tools/sparse_side.py 4 >> $O/sparse.txt 2>&1
done
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default $A/libgrem_noblk4.so $A/libgrem_bins1k.so $A/libgrem_ipt4.so $A/libgrem_bins1k_bloom.so $A/libgrem_bins1k_ipt4.so
for v in default $A/libgrem_bins1k.so $A/libgrem_ipt4.so $A/libgrem_bins1k_ipt4.so; do
  if [ $v = default ]; then PHASE_K=1 python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1
  else PHASE_K=1 GREM_LIB=$PWD/$v python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1; fi
done
