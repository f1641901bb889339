#!/bin/bash
# Round 1, third session, second call: GPU tests of the file front end and
# node statistics, then their measurements.  Run under gpurun.
set -x
O=gpurun_out/prof4
mkdir -p $O
nproc > $O/host.txt; lscpu | grep -i "model name" >> $O/host.txt; df -h /dev/shm /tmp >> $O/host.txt; free -g >> $O/host.txt
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/bench_node_stats.py papers100m > $O/node_stats.json 2> $O/node_stats.err
timeout 600 python tools/bench_file_ingest.py products 16 > $O/file_products.json 2> $O/file_products.err
timeout 900 python tools/bench_file_ingest.py papers100m 16 > $O/file_papers.json 2> $O/file_papers.err
GREM_INGEST_THREADS=1 timeout 900 python tools/bench_file_ingest.py papers100m 16 > $O/file_papers_t1.json 2> $O/file_papers_t1.err
ls -la $O
