#!/bin/bash
O=gpurun_out/r02e
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or poisoned or edge_cases or random or pinned or file' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
python -m pytest tests/test_gpu_sweep.py -s -q > $O/sweep.log 2>&1
echo "sweep rc=$?" >> $O/sweep.log
python bench.py --steps 5 --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
GREM_DEBUG_LEVELS=1 python tools/gpu_levels.py papers100m 16 > $O/timeline.txt 2>&1
