#!/bin/bash
# full ncu captures (with per-instruction source counters) of the level-0 kernels
O=gpurun_out/r02i
mkdir -p $O
python tools/gpu_bisect_once.py papers100m > $O/plain.log 2>&1 || exit 1
cap() {   # kernel regex, launch-skip, name
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
        -o $O/full_$3 python tools/gpu_bisect_once.py papers100m > $O/full_$3.log 2>&1
    ncu -i $O/full_$3.ncu-rep --page details --print-units base > $O/full_$3.txt 2>&1
    ncu -i $O/full_$3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/sass_$3.csv.gz
}
cap k_bin_scatter 4 k_bin_scatter
cap k_bin_compact 4 k_bin_compact
cap k_count_delta 6 k_count_delta
cap k_round_down 5 k_round_down
cap k_commit 3 k_commit
cap k_row_counts_bits 0 k_row_counts_bits
cap k_bfs_expand 0 k_bfs_expand
cap k_cc_link_rows 1 k_cc_link_rows
cap k_seed_map 0 k_seed_map
cap k_rank_words 0 k_rank_words
cap k_comp_keys 0 k_comp_keys
rm -f $O/*.ncu-rep
ls -la $O
