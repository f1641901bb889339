#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, one GPU).  The plain run of the
# exact same command line must exit 0 before ncu touches it.
set -u
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1700 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_init -s 2 -c 1 \
    -o gpurun_out/prof_count_init $CMD > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
