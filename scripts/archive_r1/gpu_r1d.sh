#!/bin/bash
OUT=gpurun_out/${1:-r1d}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -8 $OUT/pytest_gpu.log >> $S
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
timeout 900 python bench.py --variant parallel --steps 3 --no-cpu-baseline > $OUT/bench_simt.json 2> $OUT/bench_simt.err; echo "bench simt rc=$?" >> $S
# traffic of the dominant kernel at the bench shape (one full capture)
timeout 1200 ncu --set full --clock-control none -k regex:k7_tf32x3 -s 1 -c 1 -o $OUT/prof_k7_bench \
  python scripts/profile_one.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 2 > $OUT/prof_k7.log 2>&1; echo "ncu k7 rc=$?" >> $S
timeout 1200 ncu --set full --clock-control none -k regex:k6_sgemm -s 1 -c 1 -o $OUT/prof_k6_bench \
  python scripts/profile_one.py --variant parallel --M 32768 --N 32768 --K 8192 --reps 2 > $OUT/prof_k6.log 2>&1; echo "ncu k6 rc=$?" >> $S
