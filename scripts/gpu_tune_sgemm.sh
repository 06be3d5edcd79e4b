#!/bin/bash
OUT=gpurun_out/${1:-tune}
mkdir -p $OUT
for c in -1 0 1 2 3; do
  ELV_SGEMM_CFG=$c timeout 120 python scripts/time_variant.py --variant parallel --n 8192 >> $OUT/sgemm.jsonl 2>> $OUT/sgemm.err
done
