#!/bin/bash
O=gpurun_out/r02an
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
python tools/e2e_time.py papers100m 16 4 > $O/e2e.txt 2>&1
python bench.py --no-e2e > $O/bench_noe2e.json 2> $O/bench_noe2e.err
