#!/bin/bash
# ncu evidence (round 1, second session): run under gpurun; every profiled
# command first runs plain and must exit 0.  Outputs are kept small (<64 MiB).
set -x
O=gpurun_out/prof2
mkdir -p $O
PART=${1:-all}
if [ "$PART" = "all" ] || [ "$PART" = "launch" ]; then
python bench.py > $O/bench.json 2> $O/bench.err || exit 1
python tools/gpu_bisect_once.py papers100m > $O/bisect_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/r01b_launches_papers_level0.csv python tools/gpu_bisect_once.py papers100m > $O/l0.log 2>&1
python tools/gpu_part_once.py products 16 > $O/products_plain.log 2>&1 || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r01b_launches_products_k16.csv python tools/gpu_part_once.py products 16 > $O/prod_ncu.log 2>&1
gzip -f $O/*.csv
fi
if [ "$PART" = "all" ] || [ "$PART" = "full" ]; then
for k in k_count_delta k_bin_scatter k_bin_compact k_round_down k_round_reduce k_bin_hist; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 4 -c 1 \
      -o $O/r01b_full_$k python tools/gpu_bisect_once.py papers100m > $O/full_$k.log 2>&1
  ncu -i $O/r01b_full_$k.ncu-rep --page details --print-units base > $O/r01b_full_$k.txt 2>&1
  ncu -i $O/r01b_full_$k.ncu-rep --page raw --csv > $O/r01b_full_${k}_raw.csv 2>&1
  case $k in k_count_delta|k_bin_scatter) ;; *) rm -f $O/r01b_full_$k.ncu-rep ;; esac
done
fi
du -sh $O; ls -la $O
