#!/bin/bash
O=gpurun_out/r02o
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or poisoned or edge_cases or random or schedules' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 paper_2502_17846_b200/alt/libgrem_r01.so default
python bench.py --steps 5 > $O/bench.json 2> $O/bench.err
