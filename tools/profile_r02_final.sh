#!/bin/bash
# Round 2 final evidence (one GPU): launch list of one bench step (papers100M k=16)
# with DRAM bytes -> profiles traffic json; full captures of the top kernels of
# a level-0 bisection.  $1 = tag, $2 = source string for the traffic json.
T=${1:-r02f}
O=gpurun_out/$T
mkdir -p $O
python tools/gpu_part_once.py papers100m 16 > $O/part_plain.log 2>&1 || exit 1
GREM_NO_GRAPH=1 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_k16.csv python tools/gpu_part_once.py papers100m 16 > $O/ncu_k16.log 2>&1
python tools/ncu_summary.py $O/launches_k16.csv --traffic $O/traffic.json --source "$2" > $O/launches_k16.txt 2>&1
gzip -f $O/launches_k16.csv
cap() {   # kernel regex, launch-skip, name
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
        -o $O/full_$3 python tools/gpu_bisect_once.py papers100m > $O/full_$3.log 2>&1
    ncu -i $O/full_$3.ncu-rep --page details --print-units base > $O/full_$3.txt 2>&1
    ncu -i $O/full_$3.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/full_$3.raw.csv.gz
}
cap k_bin_scatter 4 k_bin_scatter
cap k_bin_compact 4 k_bin_compact
cap k_count_delta 6 k_count_delta
cap k_round_down 5 k_round_down
cap k_round_reduce 5 k_round_reduce
ls -la $O
