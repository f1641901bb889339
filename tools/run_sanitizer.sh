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
