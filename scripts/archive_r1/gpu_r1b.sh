#!/bin/bash
# numerics of the split-accumulator 3xTF32 kernel, GPU tests, ncu evidence
OUT=gpurun_out/${1:-r1b}
mkdir -p $OUT
timeout 300 python scripts/tf32x3_numerics.py > $OUT/num_auto.jsonl 2> $OUT/num_auto.err
ELV_TF32X3_LOLO=0 timeout 300 python scripts/tf32x3_numerics.py > $OUT/num_lolo0.jsonl 2> $OUT/num_lolo0.err
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
tail -15 $OUT/pytest_gpu.log >> $OUT/summary.txt
timeout 600 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err
# launch list of the default bench command (serialised, cold-cache: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1
# one full capture each of the two headline kernels at 8192^3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_tf32x3 -s 1 -c 1 \
  -o $OUT/prof_k7 python scripts/profile_one.py --variant parallel_tf32x3 --n 8192 --reps 2 > $OUT/prof_k7.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k56_packed -s 1 -c 1 \
  -o $OUT/prof_k6 python scripts/profile_one.py --variant parallel --n 8192 --reps 2 > $OUT/prof_k6.log 2>&1
echo done >> $OUT/summary.txt
