#!/bin/bash
# L2 residency hints A/B: interleaved timing + ncu dram bytes of the pair kernel
OUT=gpurun_out/${1:-r2_l2}; mkdir -p $OUT
for rep in 1 2; do
  for h in 0 1; do
    for enc in fp16 tf32; do
      ELV_L2_HINTS=$h ENC=$enc REPS=5 timeout 300 python scripts/gemm_once.py >> $OUT/ab.jsonl 2>> $OUT/err.log
    done
  done
done
for h in 0 1; do
  for enc in fp16 tf32; do
    ELV_L2_HINTS=$h ENC=$enc REPS=2 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum \
      --clock-control none -k regex:k7_tf32x3_pair --launch-skip 1 --launch-count 1 --csv \
      python scripts/gemm_once.py > $OUT/ncu_${enc}_h$h.csv 2>> $OUT/err.log
  done
done
timeout 300 python scripts/ladder_small.py > $OUT/ladder_small.jsonl 2>> $OUT/err.log
