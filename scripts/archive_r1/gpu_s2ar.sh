#!/bin/bash
# full evidence refresh after the 3xFP16 work: tests, sanitizers, bench, ladder, launch list
OUT=gpurun_out/${1:-s2ar}
mkdir -p $OUT
S=$OUT/summary.txt
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -n 2 $OUT/pytest_gpu.log >> $S
for t in memcheck racecheck synccheck; do
  q=""; [ $t != memcheck ] && q="--quick"
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_run.py $q > $OUT/$t.log 2>&1; echo "$t rc=$?" >> $S
done
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench ref rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1; echo "launches rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_tf32x3_pair -s 1 -c 1 \
  -o $OUT/prof_k8_bench python scripts/profile_one.py --variant parallel_fp16x3 --M 32768 --N 32768 --K 8192 --reps 2 \
  > $OUT/prof_k8.log 2>&1; echo "ncu full rc=$?" >> $S
timeout 1200 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
timeout 900 python bench.py --variant parallel --no-e2e --no-cpu-baseline > $OUT/bench_simt.json 2> $OUT/bench_simt.err; echo "bench simt rc=$?" >> $S
