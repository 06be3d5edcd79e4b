#!/bin/bash
OUT=gpurun_out/${1:-s2aj}
mkdir -p $OUT
timeout 900 python scripts/fp16x3_check.py > $OUT/numerics.jsonl 2>&1
for i in 1 2; do
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/tf32_$i.json 2> $OUT/tf32_$i.err
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline --variant parallel_fp16x3 > $OUT/fp16_$i.json 2> $OUT/fp16_$i.err
done
