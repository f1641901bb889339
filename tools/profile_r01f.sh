#!/bin/bash
# Round 1, third session, final call: full GPU suite + smoke + bench of the
# final code, node-stats hub privatisation A/B.
set -x
O=gpurun_out/prof6
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 300 python tools/bench_node_stats.py papers100m > $O/node_stats.json 2> $O/node_stats.err
GREM_NODE_STATS_NO_HUBS=1 timeout 300 python tools/bench_node_stats.py papers100m > $O/node_stats_nohubs.json 2> $O/node_stats_nohubs.err
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
ls -la $O
