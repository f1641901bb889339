#!/bin/bash
# expected_cuts / theory_curve on the GPU + the reference's support suites through the drop-in
O=gpurun_out/r02ak
mkdir -p $O
python -m pytest tests/test_curve.py -m gpu -q > $O/curve.log 2>&1; echo "rc=$?" >> $O/curve.log
python -m pytest tests/test_reference_suite.py -m gpu -q -k support -s > $O/refsuite.log 2>&1; echo "rc=$?" >> $O/refsuite.log
python tools/curve_time.py > $O/curve_time.txt 2>&1
