#!/bin/bash
OUT=gpurun_out/${1:-s2j}
mkdir -p $OUT
for bn in 64 128 256; do
  for shp in "1024 1024 1024" "1024 1024 256" "1024 1024 4096" "2048 2048 2048"; do
    set -- $shp
    ELV_TF32X3_BN=$bn timeout 120 python scripts/time_variant.py --variant parallel_tf32x3 --M $1 --N $2 --K $3 --reps 20 >> $OUT/bn_sweep.jsonl 2>&1
  done
done
for shp in "1024 1024 1024" "1024 1024 4096" "2048 2048 2048"; do
  set -- $shp
  timeout 120 python scripts/time_variant.py --variant parallel --M $1 --N $2 --K $3 --reps 20 >> $OUT/simt_small.jsonl 2>&1
done
