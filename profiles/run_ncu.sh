#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run under gpurun on ONE GPU:
#   gpurun -- bash profiles/run_ncu.sh <config> <tag>
# 1) plain bench run (must exit 0 before ncu), 2) launch list with device
# times, 3) full-set capture of the dominant kernels.
set -e
CFG=${1:-c2}
TAG=${2:-r01}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > $OUT/plain_$CFG.json 2> $OUT/plain_$CFG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches_${CFG}_${TAG}.csv $CMD > $OUT/ncu_launch_$CFG.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_nn_gemvT|k_nn_gemv|k_dense_gemv|k_spmv" -s 40 -c 4 \
    -o $OUT/prof_${CFG}_${TAG} $CMD > $OUT/ncu_full_$CFG.log 2>&1
echo done
