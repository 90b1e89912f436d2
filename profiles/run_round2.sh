#!/bin/bash
# Round-2 measurement set (one GPU, under gpurun): the default bench line (c5),
# the c2 / c3 bench lines, the reference arm, then the c5 ncu captures
# (profiles/run_ncu_c5.sh: launch list + one full-set capture of the dominant
# kernels on the real c5 factors; gpurun only profiles commands whose plain
# run ends within 300 s, see prof_solve.py).
#   gpurun -- bash profiles/run_round2.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python bench.py --verbose > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err
echo "bench c5 rc=$?"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
echo "bench c2 rc=$?"
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err
echo "bench c3 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref_c5_$TAG.json 2> $OUT/bench_ref_c5_$TAG.err
echo "reference arm rc=$?"
bash profiles/run_ncu_c5.sh $TAG
