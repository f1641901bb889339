#!/bin/bash
O=gpurun_out/r02bg
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
