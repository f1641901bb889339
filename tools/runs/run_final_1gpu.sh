#!/bin/bash
# Round-2 final evidence on one B200.  $1 = source tag for the traffic json
O=gpurun_out/final1
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 paper_2502_17846_b200/alt/libgrem_r01.so default env:GREM_NO_PDL=1 env:GREM_NO_PREFETCH=1
python tools/gpu_time.py friendster 256 6 > $O/friendster.txt 2>&1
python tools/gpu_time.py friendster 16 4 >> $O/friendster.txt 2>&1
python tools/gpu_time.py products 16 6 >> $O/friendster.txt 2>&1
GREM_DEBUG_LEVELS=1 python tools/gpu_levels.py papers100m 16 > $O/timeline.txt 2>&1
bash tools/profile_r02_final.sh final1/prof "$1" > $O/prof.log 2>&1
