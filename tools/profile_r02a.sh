#!/bin/bash
# Round 2: per-bisection timeline, launch list with DRAM bytes of one
# papers100M-shaped k=16 partition (the bench step).  Run under gpurun.
set -x
O=gpurun_out/r02p
mkdir -p $O
python tools/gpu_part_once.py papers100m 16 > $O/part_plain.log 2>&1 || exit 1
GREM_DEBUG_LEVELS=1 python tools/gpu_levels.py papers100m 16 > $O/timeline.txt 2>&1
GREM_DEBUG_LEVELS=1 GREM_SERIAL_SIBLINGS=1 python tools/gpu_levels_phases.py papers100m 16 > $O/levels_phases.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_k16.csv python tools/gpu_part_once.py papers100m 16 > $O/ncu_k16.log 2>&1
python tools/ncu_summary.py $O/launches_k16.csv --traffic $O/traffic.json --source "$1" > $O/launches_k16.txt 2>&1
gzip -f $O/*.csv
ls -la $O
