#!/bin/bash
OUT=gpurun_out/${1:-grp}
mkdir -p $OUT
S=$OUT/summary.txt
for r in 1 2; do for g in 8 16 4 32; do
  echo "== group=$g rep $r" >> $S
  ELV_TILE_GROUP=$g timeout 300 python scripts/time_variant.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 3 >> $S 2>>$OUT/err.txt
done; done
for g in 8 16 4; do
  echo "== ncu group=$g" >> $S
  ELV_TILE_GROUP=$g timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:k7_tf32x3 -c 1 \
     python scripts/profile_one.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 1 2>&1 | grep -E "dram__bytes_read|gpu__time|hit_rate" >> $S
done
