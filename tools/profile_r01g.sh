#!/bin/bash
# Round 1, last session: full capture of k_count_delta after the
# four-loads-in-flight change, plus the level-0 launch list.  Run under gpurun.
set -x
O=gpurun_out/prof12
mkdir -p $O
python tools/gpu_bisect_once.py papers100m > $O/bisect_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/r01d_launches_papers_level0.csv python tools/gpu_bisect_once.py papers100m > $O/l0.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count_delta --launch-skip 4 -c 1 \
    -o $O/r01d_full_k_count_delta python tools/gpu_bisect_once.py papers100m > $O/full_cd.log 2>&1
ncu -i $O/r01d_full_k_count_delta.ncu-rep --page details --print-units base > $O/r01d_full_k_count_delta.txt 2>&1
gzip -f $O/*.csv
ls -la $O
