#!/bin/bash
OUT=gpurun_out/${1:-raster}
mkdir -p $OUT
S=$OUT/summary.txt
ELV_TF32X3_PAIR=32 timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "tf32x3" -p no:cacheprovider > $OUT/pytest_pair32.log 2>&1; echo "pair32 pytest rc=$?" >> $S
tail -3 $OUT/pytest_pair32.log >> $S
for cfg in "0 16" "0 8" "0 32" "0 4" "16 8" "16 4" "16 16" "32 8" "32 4" "32 16"; do
  set -- $cfg
  echo "== pair=$1 group=$2" >> $S
  ELV_TF32X3_PAIR=$1 ELV_TILE_GROUP=$2 timeout 300 python scripts/time_variant.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 3 >> $S 2>>$OUT/err.txt
  ELV_TF32X3_PAIR=$1 ELV_TILE_GROUP=$2 timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:k7_tf32x3 -c 1 \
     python scripts/profile_one.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 1 2>&1 | grep -E "dram__bytes_read|gpu__time|hit_rate" >> $S
done
