#!/bin/bash
O=gpurun_out/r02l
mkdir -p $O
python -m pytest tests -m gpu -x -q -k 'golden or binned or hub or poisoned or edge_cases or random or schedules' > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
for v in paper_2502_17846_b200/alt/libgrem_r01.so default; do
    if [ $v = default ]; then python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1;
    else GREM_LIB=$PWD/$v python tools/phase_ab.py papers100m 16 >> $O/phases.txt 2>&1; fi
done
bash tools/ab_time.sh $O/ab.txt papers100m 16 8 paper_2502_17846_b200/alt/libgrem_r01.so default
