#!/bin/bash
# full GPU suite on the current build + A/B (papers k=16, friendster k=256) vs the previous commit
O=gpurun_out/r02al
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default paper_2502_17846_b200/alt/libgrem_head.so
bash tools/ab_time.sh $O/ab_f256.txt friendster 256 3 default paper_2502_17846_b200/alt/libgrem_head.so
