#!/bin/bash
OUT=gpurun_out/${1:-r2_l2b}; mkdir -p $OUT
for h in 0 1; do
  for g in 8 16; do
    for enc in fp16 tf32; do
      ELV_TILE_GROUP=$g ELV_L2_HINTS=$h ENC=$enc REPS=2 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum \
        --clock-control none -k regex:k7_tf32x3_pair --launch-skip 1 --launch-count 1 --csv \
        python scripts/gemm_once.py > $OUT/ncu_${enc}_h${h}_g$g.csv 2>> $OUT/err.log
    done
  done
done
