#!/bin/bash
O=gpurun_out/r02ay
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python -m pytest tests/test_gpu_sweep.py -m gpu -s -q > $O/sweep.log 2>&1; echo "rc=$?" >> $O/sweep.log
