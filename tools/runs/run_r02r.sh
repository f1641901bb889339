#!/bin/bash
O=gpurun_out/r02r
mkdir -p $O
GREM_DEBUG_MEM=1 python tools/gpu_time.py friendster 256 5 > $O/friendster256.txt 2> $O/friendster256.err
echo "rc=$?" >> $O/friendster256.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_level0.csv python tools/gpu_bisect_once.py papers100m > $O/l0.log 2>&1
python tools/ncu_summary.py $O/launches_level0.csv > $O/launches_level0.txt 2>&1
gzip -f $O/*.csv
