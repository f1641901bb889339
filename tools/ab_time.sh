#!/bin/bash
# A/B of library builds / env switches inside one gpurun call (same box, interleaved twice):
# tools/ab_time.sh OUT SHAPE K REPS variant...   variant: "default" (in-tree build), a .so path, or env:VAR=VAL
OUT=$1; SHAPE=$2; K=$3; REPS=$4; shift 4
for round in 1 2; do
    for v in "$@"; do
        echo "[variant $v]" >> $OUT
        case "$v" in
            default) python tools/gpu_time.py $SHAPE $K $REPS >> $OUT 2>&1 ;;
            env:*) env ${v#env:} python tools/gpu_time.py $SHAPE $K $REPS >> $OUT 2>&1 ;;
            *) GREM_LIB=$PWD/$v python tools/gpu_time.py $SHAPE $K $REPS >> $OUT 2>&1 ;;
        esac
    done
done
