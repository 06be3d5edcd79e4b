#!/bin/bash
OUT=gpurun_out/${1:-pairws}
mkdir -p $OUT
S=$OUT/summary.txt
ELV_TF32X3_PAIR=32 timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "tf32x3" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest pair32 rc=$?" >> $S
for r in 1 2; do for cfg in "0 16" "16 8" "16 16" "32 8" "32 16"; do
  set -- $cfg
  echo "== pair=$1 group=$2" >> $S
  ELV_TF32X3_PAIR=$1 ELV_TILE_GROUP=$2 timeout 300 python scripts/time_variant.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 3 >> $S 2>>$OUT/err.txt
done; done
for cfg in "16 16" "32 16"; do
  set -- $cfg
  echo "== ncu pair=$1 group=$2" >> $S
  ELV_TF32X3_PAIR=$1 ELV_TILE_GROUP=$2 timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:k7_tf32x3 -c 1 \
     python scripts/profile_one.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 1 2>&1 | grep -E "dram__bytes_read|gpu__time" >> $S
done
