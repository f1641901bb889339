#!/bin/bash
# Round 1, third session, third call: e2e (page-locked host edges) vs
# device-resident partition, copy-stream priority A/B, then the bench line.
set -x
O=gpurun_out/prof5
mkdir -p $O
timeout 600 python -m pytest tests/test_theory.py tests/test_gpu_parity.py -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/bench_node_stats.py papers100m > $O/node_stats.json 2> $O/node_stats.err
GREM_NODE_STATS_UNPACKED=1 timeout 300 python tools/bench_node_stats.py papers100m > $O/node_stats_unpacked.json 2> $O/node_stats_unpacked.err
timeout 600 python tools/gpu_levels_e2e.py papers100m 16 > $O/e2e_hi.log 2>&1
GREM_COPY_PRIO_LOW=1 timeout 600 python tools/gpu_levels_e2e.py papers100m 16 > $O/e2e_lo.log 2>&1
GREM_DEBUG_LEVELS=1 timeout 600 python tools/gpu_levels_e2e.py papers100m 16 > $O/e2e_levels.log 2>&1
timeout 900 python tools/bench_file_ingest.py papers100m 16 > $O/file_papers.json 2> $O/file_papers.err
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
ls -la $O
