#!/bin/bash
O=gpurun_out/r02q
mkdir -p $O
python tools/gpu_time.py friendster 256 5 > $O/friendster.txt 2>&1
GREM_DEBUG_MEM=1 python tools/gpu_time.py friendster 128 4 > $O/friendster128_mem.txt 2>&1
python -m pytest tests/test_gpu_sweep.py -s -q > $O/sweep.log 2>&1
python -m pytest tests -m gpu -x -q -k 'golden or schedules' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
