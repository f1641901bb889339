#!/bin/bash
O=gpurun_out/r02x
mkdir -p $O
for v in "GREM_NO_PREFETCH=1" "GREM_SPAWN_FREE=0.0" "GREM_SPAWN_FREE=0.99" "GREM_MAX_CTX=1000" "GREM_NONE=1"; do
    env $v python tools/gpu_time.py friendster 256 5 >> $O/f256.txt 2>> $O/f256_$v.err
    echo "$v rc=$?" >> $O/f256.txt
done
