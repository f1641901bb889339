#!/bin/bash
O=gpurun_out/r02ax
mkdir -p $O
python tools/gpu_part_once.py papers100m 4 > $O/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_edges -c 1 \
    -o $O/full_k_split_edges python tools/gpu_part_once.py papers100m 4 > $O/full.log 2>&1
ncu -i $O/full_k_split_edges.ncu-rep --page details --print-units base > $O/full_k_split_edges.txt 2>&1
ncu -i $O/full_k_split_edges.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/sass_k_split_edges.csv.gz
rm -f $O/full_k_split_edges.ncu-rep
