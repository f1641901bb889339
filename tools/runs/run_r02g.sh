#!/bin/bash
O=gpurun_out/r02g
mkdir -p $O
SUBTREE_PROFILE=0 python tools/gpu_subtree.py 1 > $O/subtree1_noprof.txt 2>&1
SUBTREE_PROFILE=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --graph-profiling node --csv \
    --log-file $O/launches_sparse1_warm.csv python tools/gpu_subtree.py 1 > $O/sparse1_ncu.log 2>&1
python tools/ncu_summary.py $O/launches_sparse1_warm.csv > $O/launches_sparse1_warm.txt 2>&1
gzip -f $O/*.csv
