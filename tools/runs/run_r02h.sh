#!/bin/bash
O=gpurun_out/r02h
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or poisoned or edge_cases or random or schedules or kernels or variants' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
SUBTREE_PROFILE=0 python tools/gpu_subtree.py 1 > $O/subtree1_skip.txt 2>&1
GREM_BUNDLE_NO_SKIP=1 SUBTREE_PROFILE=0 python tools/gpu_subtree.py 1 > $O/subtree1_noskip.txt 2>&1
python bench.py --steps 5 --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
GREM_BUNDLE_NO_SKIP=1 python bench.py --steps 5 --no-cpu --no-e2e > $O/bench_noskip.json 2> $O/bench_noskip.err
for spec in k_count_delta:70:cd k_round_down:80:rd k_bundle_sim:40:sim; do
    IFS=: read re skip name <<< "$spec"
    SUBTREE_PROFILE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$re --launch-skip $skip -c 1 \
        -o $O/sparse_full_$name python tools/gpu_subtree.py 1 > $O/sparse_full_$name.log 2>&1
    ncu -i $O/sparse_full_$name.ncu-rep --page details --print-units base > $O/sparse_full_$name.txt 2>&1
    ncu -i $O/sparse_full_$name.ncu-rep --page source --csv 2>/dev/null | gzip > $O/sparse_full_$name.source.csv.gz
done
