#!/bin/bash
# c5 ncu captures under gpurun's rule that the profiled command first runs to
# completion without ncu in under 300 s: profiles/prof_solve.py c5 reference 1e-2
# (real c5 local factors, coarse space and K0; W of the real shape from
# loosely converged inner PCGs — see prof_solve.py).
#   gpurun -- bash profiles/run_ncu_c5.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
CMD="python profiles/prof_solve.py c5 reference 1e-2"
timeout 290 $CMD > $OUT/plain_c5_$TAG.log 2>&1
echo "plain rc=$?"; tail -1 $OUT/plain_c5_$TAG.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches_c5_$TAG.csv $CMD > $OUT/ncu_launch_c5_$TAG.log 2>&1
echo "ncu launch rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_nn_fused|k_dense_gemvT_part|k_dense_gemv" -s 6 -c 6 \
    -o $OUT/prof_c5_$TAG $CMD > $OUT/ncu_full_c5_$TAG.log 2>&1
echo "ncu full rc=$?"
