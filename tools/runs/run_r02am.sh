#!/bin/bash
# e2e from pinned host memory: id checks on their own stream vs the committed build
O=gpurun_out/r02am
mkdir -p $O
for v in default alt; do
  for r in 1 2; do
    if [ $v = alt ]; then GREM_LIB=$PWD/paper_2502_17846_b200/alt/libgrem_head.so python tools/e2e_time.py papers100m 16 4 >> $O/e2e.txt 2>&1
    else python tools/e2e_time.py papers100m 16 4 >> $O/e2e.txt 2>&1; fi
  done
done
python -m pytest tests -m gpu -x -q -k 'ingest or file or pinned or host or bad' > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
