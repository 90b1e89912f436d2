#!/bin/bash
# Round-end measurement set (one GPU, under gpurun): default bench line, the
# ncu launch list of the same command's timed region, one full-set capture of
# the solve kernels, then the c3 and c5 bench lines.
#   gpurun -- bash profiles/run_round.sh <tag>
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err; echo "bench c2 rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_bench_c2_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_nn_fused|k_bs_gemvT|k_prolong_sum|k_spmv_aplus|k_pcg_spmv_dot_p|k_prolong_nn|k_coarse_solve" -c 8 \
    -o $OUT/prof_c2_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
timeout 900 python bench.py --config c3 --steps 5 > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err; echo "bench c3 rc=$?"
AWG_VERBOSE=1 timeout 2000 python bench.py --config c5 --steps 3 > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err; echo "bench c5 rc=$?"
