#!/bin/bash
# labels copy-out overlapped with the final cut pass: e2e A/B vs HEAD + GPU suite
O=gpurun_out/r02bc
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  python tools/e2e_time.py papers100m 16 5 >> $O/e2e.txt 2>&1
  GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_head.so python tools/e2e_time.py papers100m 16 5 >> $O/e2e.txt 2>&1
done
