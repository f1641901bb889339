#!/bin/bash
# new scatter footprint (1024 bins + hub prefilter + odd carry stride): full GPU suite, A/B vs HEAD, bench
O=gpurun_out/r02as
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default paper_2502_17846_b200/alt/libgrem_head.so
bash tools/ab_time.sh $O/ab_f.txt friendster 16 4 default paper_2502_17846_b200/alt/libgrem_head.so
PHASE_K=1 python tools/phase_ab.py papers100m 16 > $O/phases.txt 2>&1
python bench.py > $O/bench.json 2> $O/bench.err
