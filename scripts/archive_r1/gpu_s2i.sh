#!/bin/bash
# evidence set: tests, ladder, bench (+ref arm), launch list, ncu full of K7 (bench shape) and small kernels
OUT=gpurun_out/${1:-s2i}
mkdir -p $OUT
S=$OUT/summary.txt
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -4 $OUT/pytest_gpu.log >> $S
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
timeout 900 python bench.py --variant parallel --steps 3 --no-cpu-baseline > $OUT/bench_simt.json 2> $OUT/bench_simt.err; echo "bench simt rc=$?" >> $S
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench ref rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1; echo "launches rc=$?" >> $S
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k7_tf32x3 -s 1 -c 1 -o $OUT/prof_k7_bench \
  python scripts/profile_one.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 2 > $OUT/prof_k7.log 2>&1; echo "ncu k7 rc=$?" >> $S
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k7_tf32x3|k6_sgemm_small|k_split_ab" -s 3 -c 3 -o $OUT/prof_small \
  python scripts/profile_one.py --variant parallel_tf32x3 --n 1024 --reps 3 > $OUT/prof_small.log 2>&1; echo "ncu small rc=$?" >> $S
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k6_sgemm_small" -s 1 -c 1 -o $OUT/prof_small6 \
  python scripts/profile_one.py --variant parallel --n 1024 --reps 3 > $OUT/prof_small6.log 2>&1; echo "ncu small6 rc=$?" >> $S
