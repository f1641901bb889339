#!/bin/bash
O=gpurun_out/r02ao
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
