#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small partitions (one GPU)
O=gpurun_out/r02s
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for shape in tiny:4 arxiv:8; do
    IFS=: read s k <<< "$shape"
    timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/gpu_part_once.py $s $k > $O/memcheck_${s}_k$k.txt 2>&1
    echo "exit=$?" >> $O/memcheck_${s}_k$k.txt
done
timeout 1500 $CS --tool racecheck --error-exitcode 9 python tools/gpu_part_once.py tiny 4 > $O/racecheck_tiny_k4.txt 2>&1
echo "exit=$?" >> $O/racecheck_tiny_k4.txt
timeout 1200 $CS --tool synccheck --error-exitcode 9 python tools/gpu_part_once.py tiny 4 > $O/synccheck_tiny_k4.txt 2>&1
echo "exit=$?" >> $O/synccheck_tiny_k4.txt
GREM_FORCE_BINNING=1 GREM_HUB_MIN_CHUNK=1000 timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/gpu_part_once.py arxiv 8 > $O/memcheck_arxiv_k8_binned_hubs.txt 2>&1
echo "exit=$?" >> $O/memcheck_arxiv_k8_binned_hubs.txt
GREM_FORCE_BINNING=1 GREM_HUB_MIN_CHUNK=1000 timeout 1500 $CS --tool racecheck --error-exitcode 9 python tools/gpu_part_once.py tiny 4 > $O/racecheck_tiny_k4_binned_hubs.txt 2>&1
echo "exit=$?" >> $O/racecheck_tiny_k4_binned_hubs.txt
# early-round captures in the level-1 sparse bisection (after the level-0 bisection's launches)
for spec in k_count_delta:46:cd_r2 k_round_down:55:rd_r2 k_bundle_sim:1:sim_r2 k_round_reduce:55:rr_r2; do
    IFS=: read re skip name <<< "$spec"
    SUBTREE_PROFILE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$re --launch-skip $skip -c 1 \
        -o $O/sparse_full_$name python tools/gpu_subtree.py 1 > $O/sparse_full_$name.log 2>&1
    ncu -i $O/sparse_full_$name.ncu-rep --page details --print-units base > $O/sparse_full_$name.txt 2>&1
    ncu -i $O/sparse_full_$name.ncu-rep --page source --csv 2>/dev/null | gzip > $O/sparse_full_$name.source.csv.gz
    rm -f $O/sparse_full_$name.ncu-rep
done
GREM_DEBUG_LEVELS=1 python tools/gpu_levels_e2e.py papers100m 16 > $O/e2e_timeline.txt 2>&1
