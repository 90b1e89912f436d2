#!/bin/bash
# Round-2 measurement set (one GPU, under gpurun): the default bench line (c5),
# the ncu launch list of the same command's timed region, one full-set capture
# of the dominant kernel (k_nn_fused) in that run, the c2 / c3 bench lines and
# the reference arm.  Every ncu command runs only after the same command exited
# 0 without ncu (B200_PROFILING.md).
#   gpurun -- bash profiles/run_round2.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python bench.py --steps 5 --warmup 3 > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err
echo "bench c5 rc=$?"
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file $OUT/launches_bench_c5_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > $OUT/ncu_launch_c5_$TAG.log 2>&1
echo "ncu launch rc=$?"
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_nn_fused|k_dense_gemvT_part|k_dense_gemv" -c 3 \
    -o $OUT/prof_c5_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_c5_$TAG.log 2>&1
echo "ncu full rc=$?"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
echo "bench c2 rc=$?"
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err
echo "bench c3 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref_c5_$TAG.json 2> $OUT/bench_ref_c5_$TAG.err
echo "reference arm rc=$?"
VERBOSE=2 timeout 900 python profiles/setup_only.py c5 > $OUT/setup_c5_$TAG.json 2> $OUT/setup_c5_trace_$TAG.txt
echo "setup trace rc=$?"
