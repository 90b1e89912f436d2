#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run under gpurun on ONE GPU:
#   gpurun -- bash profiles/run_ncu.sh <config> <tag>
# Only the solve is profiled (profiles/prof_solve.py brackets one PCG solve
# with cudaProfilerStart/Stop).  1) plain run (must exit 0 first), 2) launch
# list with device times, 3) full-set capture of the dominant kernels.
set -e
CFG=${1:-c2}
TAG=${2:-r01}
OUT=gpurun_out
mkdir -p $OUT
CMD="python profiles/prof_solve.py $CFG"
$CMD > $OUT/plain_$CFG.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $OUT/launches_${CFG}_${TAG}.csv $CMD > $OUT/ncu_launch_$CFG.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_nn_fused|k_nn_gemvT|k_nn_gemv|k_dense_gemv|k_spmv|k_prolong|k_bs_gemvT" -s 10 -c 9 \
    -o $OUT/prof_${CFG}_${TAG} $CMD > $OUT/ncu_full_$CFG.log 2>&1
echo done
