#!/bin/bash
# final-build evidence after the green-context default change
O=gpurun_out/r02ad
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 default paper_2502_17846_b200/alt/libgrem_r01.so
