#!/bin/bash
# the papers100M level-1 sparse side as a standalone bisection: timing, phases, ncu of its round kernels
O=gpurun_out/r02p3
mkdir -p $O
python tools/sparse_side.py 4 > $O/time.txt 2>&1 || exit 1
PHASES=1 python tools/sparse_side.py 2 > $O/phases.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python tools/sparse_side.py 1 > $O/ncu_list.log 2>&1
python tools/ncu_summary.py $O/launches.csv > $O/launches.txt 2>&1; gzip -f $O/launches.csv
cap() {   # kernel regex, launch-skip, name
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
        -o $O/full_$3 python tools/sparse_side.py 1 > $O/full_$3.log 2>&1
    ncu -i $O/full_$3.ncu-rep --page details --print-units base > $O/full_$3.txt 2>&1
    ncu -i $O/full_$3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/sass_$3.csv.gz
    rm -f $O/full_$3.ncu-rep
}
cap k_bundle_sim 40 k_bundle_sim
cap k_bundle_chain 40 k_bundle_chain
cap k_bundle_final 40 k_bundle_final
cap k_bundle_fix 40 k_bundle_fix
cap k_round_down 40 k_round_down
cap k_round_reduce 40 k_round_reduce
cap k_count_delta 40 k_count_delta
cap k_round_start 40 k_round_start
cap k_scan_top_gated 40 k_scan_top_gated
