#!/bin/bash
# Quick A/B under gpurun: parity subset, bench (default build and any
# alternative builds in paper_2502_17846_b200/alt/), level-0 launch list.
# usage: tools/perf_check.sh TAG
T=${1:-pc}
O=gpurun_out/$T
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or poisoned or edge_cases or random or schedules' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
python bench.py --steps 5 --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
for lib in paper_2502_17846_b200/alt/*.so; do
    [ -e "$lib" ] || continue
    b=$(basename $lib .so)
    GREM_LIB=$PWD/$lib python bench.py --steps 5 --no-cpu --no-e2e > $O/bench_$b.json 2> $O/bench_$b.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_level0.csv python tools/gpu_bisect_once.py papers100m > $O/l0.log 2>&1
python tools/ncu_summary.py $O/launches_level0.csv > $O/launches_level0.txt 2>&1
gzip -f $O/*.csv
GREM_DEBUG_BUNDLE=1 python tools/gpu_subtree.py 1 > $O/subtree1_bundle.txt 2>&1
