#!/bin/bash
# ncu evidence for round 1 (run under gpurun; each command first runs plain)
set -x
make -s -C paper_2502_17846_b200/csrc >/dev/null 2>&1
O=gpurun_out/prof
mkdir -p $O
python tools/gpu_bisect_once.py papers100m > $O/bisect_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01_launches_papers_level0.csv \
    python tools/gpu_bisect_once.py papers100m > $O/l0.log 2>&1
python bench.py --workload products --steps 1 --warmup 0 --no-e2e --no-cpu > $O/products_plain.log 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01_launches_products_k16.csv \
    python bench.py --workload products --steps 1 --warmup 0 --no-e2e --no-cpu > $O/prod_ncu.log 2>&1
for k in k_count_delta k_bin_apply k_bin_scatter k_round_reduce k_round_down; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 \
      -o $O/r01_full_$k python tools/gpu_bisect_once.py papers100m > $O/full_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bundle_sim --launch-skip 200 -c 1 \
    -o $O/r01_full_k_bundle_sim python tools/gpu_subtree.py 1 > $O/full_bundle.log 2>&1
ls -la $O
