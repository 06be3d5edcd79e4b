#!/bin/bash
OUT=gpurun_out/${1:-pair}
mkdir -p $OUT
S=$OUT/summary.txt
ELV_TF32X3_PAIR=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "tf32x3" -p no:cacheprovider > $OUT/pytest_pair.log 2>&1; echo "pair pytest rc=$?" >> $S
tail -8 $OUT/pytest_pair.log >> $S
for pr in 0 1; do
  ELV_TF32X3_PAIR=$pr timeout 120 python scripts/time_variant.py --variant parallel_tf32x3 --n 8192 >> $OUT/time.jsonl 2>>$OUT/time.err
  ELV_TF32X3_PAIR=$pr timeout 300 python scripts/time_variant.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 3 >> $OUT/time.jsonl 2>>$OUT/time.err
done
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -8 $OUT/pytest_gpu.log >> $S
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
ELV_TF32X3_PAIR=1 timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_pair.json 2> $OUT/bench_pair.err; echo "bench pair rc=$?" >> $S
