#!/bin/bash
O=gpurun_out/r02ab
mkdir -p $O
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 default env:GREM_BUNDLE_K=8 env:GREM_BUNDLE_K=12 env:GREM_BUNDLE_K=48
