#!/bin/bash
O=gpurun_out/r02av
mkdir -p $O
python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
