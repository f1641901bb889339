#!/bin/bash
O=gpurun_out/r02y
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
python tools/gpu_time.py friendster 256 8 > $O/f256.txt 2>&1
echo "rc=$?" >> $O/f256.txt
python tools/gpu_time.py papers100m 16 10 > $O/papers.txt 2>&1
