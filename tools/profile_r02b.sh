#!/bin/bash
# Round 2: full ncu captures of the level-0 top kernels (papers100M-shaped,
# one level-0 bisection, tools/gpu_bisect_once.py), after the same command
# exited 0 without ncu, plus the level-0 launch list with DRAM bytes.
# Run under gpurun:  CAPS="k_round_down:0:round_down_r1 ..." tools/profile_r02b.sh TAG
set -x
T=${1:-r02}
O=gpurun_out/$T
mkdir -p $O
python tools/gpu_bisect_once.py papers100m > $O/bisect_plain.log 2>&1 || exit 1
cap() {   # kernel regex, launch-skip, name
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
        -o $O/full_$3 python tools/gpu_bisect_once.py papers100m > $O/full_$3.log 2>&1
    ncu -i $O/full_$3.ncu-rep --page details --print-units base > $O/full_$3.txt 2>&1
    ncu -i $O/full_$3.ncu-rep --page source --csv > $O/full_$3.source.csv 2>&1
}
for spec in $CAPS; do
    IFS=: read re skip name <<< "$spec"
    cap "$re" "$skip" "$name"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_level0.csv python tools/gpu_bisect_once.py papers100m > $O/l0.log 2>&1
python tools/ncu_summary.py $O/launches_level0.csv > $O/launches_level0.txt 2>&1
gzip -f $O/*.csv
ls -la $O
