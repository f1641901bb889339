#!/bin/bash
O=gpurun_out/r02f
mkdir -p $O
python -m pytest tests/test_gpu_sweep.py -s -q > $O/sweep.log 2>&1
echo "sweep rc=$?" >> $O/sweep.log
python bench.py --steps 5 --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
GREM_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_sparse1.csv python tools/gpu_subtree.py 1 > $O/sparse1_ncu.log 2>&1
python tools/ncu_summary.py $O/launches_sparse1.csv > $O/launches_sparse1.txt 2>&1
gzip -f $O/*.csv
