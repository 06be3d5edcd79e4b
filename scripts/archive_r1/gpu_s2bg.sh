#!/bin/bash
OUT=gpurun_out/${1:-s2bg}
mkdir -p $OUT
for i in 1 2; do
  for plan in grid grow; do
    ELV_HOST_PLAN=$plan timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/bench_${plan}_$i.json 2> $OUT/bench_${plan}_$i.err
  done
done
