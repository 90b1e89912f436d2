set -e
OUT=gpurun_out
python profiles/op_times.py c2 > $OUT/op_times_c2.json 2> $OUT/op_times_c2.err
python profiles/prof_solve.py c2 > $OUT/plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv --log-file $OUT/launches_c2_warm.csv python profiles/prof_solve.py c2 > $OUT/ncu_warm.log 2>&1
echo done
