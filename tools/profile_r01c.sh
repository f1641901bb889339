#!/bin/bash
# Round 1, third session: re-validate the current code on one B200 and
# refresh the evidence (tests, smoke, both bench arms, launch lists, one
# full capture of the roofline kernel).  Run under gpurun.
set -x
O=gpurun_out/prof3
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err || exit 1
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
python tools/gpu_bisect_once.py papers100m > $O/bisect_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/r01c_launches_papers_level0.csv python tools/gpu_bisect_once.py papers100m > $O/l0.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r01c_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $O/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count_delta --launch-skip 4 -c 1 \
    -o $O/r01c_full_k_count_delta python tools/gpu_bisect_once.py papers100m > $O/full_cd.log 2>&1
ncu -i $O/r01c_full_k_count_delta.ncu-rep --page details --print-units base > $O/r01c_full_k_count_delta.txt 2>&1
gzip -f $O/*.csv
du -sh $O; ls -la $O
