#!/bin/bash
OUT=gpurun_out/${1:-tune}
mkdir -p $OUT
for c in 0 2 4; do
  ELV_SGEMM_CFG=$c timeout 120 python scripts/time_variant.py --variant parallel --n 8192 >> $OUT/sgemm.jsonl 2>> $OUT/sgemm.err
  ELV_SGEMM_CFG=$c timeout 300 python scripts/time_variant.py --variant parallel --M 32768 --N 32768 --K 8192 --reps 2 >> $OUT/sgemm.jsonl 2>> $OUT/sgemm.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k6_sgemm_8x16 -s 1 -c 1 \
  -o $OUT/prof_k6_8x16 env ELV_SGEMM_CFG=4 python scripts/profile_one.py --variant parallel --n 8192 --reps 2 > $OUT/prof.log 2>&1
