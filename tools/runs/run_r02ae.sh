#!/bin/bash
# A/B of scheduling knobs on papers100M k=16
O=gpurun_out/r02ae
mkdir -p $O
bash tools/ab_time.sh $O/ab.txt papers100m 16 6 default env:GREM_GRAPH_REPLAYS=2 env:GREM_BUNDLE_K=12 env:GREM_BUNDLE_K=48 env:GREM_PRIO=0 env:GREM_PRIO=2 env:GREM_DEFER=1 env:GREM_SERIAL_SIBLINGS=1
