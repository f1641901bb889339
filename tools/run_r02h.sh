#!/bin/bash
O=gpurun_out/r02h
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or poisoned or edge_cases or random or schedules or kernels or variants' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
SUBTREE_PROFILE=0 python tools/gpu_subtree.py 1 > $O/subtree1_skip.txt 2>&1
GREM_BUNDLE_NO_SKIP=1 SUBTREE_PROFILE=0 python tools/gpu_subtree.py 1 > $O/subtree1_noskip.txt 2>&1
python bench.py --steps 5 --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
GREM_BUNDLE_NO_SKIP=1 python bench.py --steps 5 --no-cpu --no-e2e > $O/bench_noskip.json 2> $O/bench_noskip.err
