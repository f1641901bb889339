#!/bin/bash
# Final evidence for the current build: launch lists (k=16 step and one level-0
# bisection) with DRAM bytes -> traffic json; full captures of the top level-0 kernels.
# $1 = tag, $2 = commit for the source strings
T=${1:-r02g}; C=${2:-HEAD}
O=gpurun_out/$T
mkdir -p $O
python tools/gpu_part_once.py papers100m 16 > $O/part_plain.log 2>&1 || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
GREM_NO_GRAPH=1 timeout 1500 ncu --metrics $M --clock-control none --csv --log-file $O/launches_k16.csv \
    python tools/gpu_part_once.py papers100m 16 > $O/ncu_k16.log 2>&1
python tools/ncu_summary.py $O/launches_k16.csv --traffic $O/traffic_k16.json \
    --source "profiles/r02_final_launches_k16.txt: ncu launch list of one papers100M k=16 partition, commit $C" > $O/launches_k16.txt 2>&1
gzip -f $O/launches_k16.csv
GREM_NO_GRAPH=1 timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_l0.csv \
    python tools/gpu_bisect_once.py papers100m > $O/ncu_l0.log 2>&1
python tools/ncu_summary.py $O/launches_l0.csv --traffic $O/traffic_l0.json \
    --source "profiles/r02_launches_level0.txt: average DRAM bytes per launch over one papers100M level-0 bisection (all its launches of the kernel, cold caches), commit $C" > $O/launches_l0.txt 2>&1
gzip -f $O/launches_l0.csv
python - "$O" <<'PY'
import json, sys
o = sys.argv[1]
l0 = json.load(open(f"{o}/traffic_l0.json")); k16 = json.load(open(f"{o}/traffic_k16.json"))
l0.pop("step", None); l0["step"] = k16["step"]
json.dump(l0, open(f"{o}/traffic.json", "w"), indent=1, sort_keys=True)
PY
cap() {   # kernel regex, launch-skip, name
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
        -o $O/full_$3 python tools/gpu_bisect_once.py papers100m > $O/full_$3.log 2>&1
    ncu -i $O/full_$3.ncu-rep --page details --print-units base > $O/full_$3.txt 2>&1
    ncu -i $O/full_$3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/sass_$3.csv.gz
}
cap k_bin_scatter 4 k_bin_scatter
cap k_bin_compact 4 k_bin_compact
cap k_count_delta 6 k_count_delta
cap k_round_down 5 k_round_down
cap k_round_reduce 5 k_round_reduce
rm -f $O/full_k_bin_compact.ncu-rep $O/full_k_count_delta.ncu-rep $O/full_k_round_down.ncu-rep $O/full_k_round_reduce.ncu-rep
ls -la $O
