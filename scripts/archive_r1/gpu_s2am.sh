#!/bin/bash
# evidence set with the 3xFP16 default
OUT=gpurun_out/${1:-s2am}
mkdir -p $OUT
S=$OUT/summary.txt
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -n 3 $OUT/pytest_gpu.log >> $S
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1; echo "launches rc=$?" >> $S
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k7_tf32x3_pair -s 1 -c 1 -o $OUT/prof_k7_fp16 \
  python scripts/profile_one.py --variant parallel_fp16x3 --M 32768 --N 32768 --K 8192 --reps 2 > $OUT/prof_k7.log 2>&1; echo "ncu k7fp16 rc=$?" >> $S
