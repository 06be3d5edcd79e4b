#!/bin/bash
# ncu --set full of the 1-CTA tcgen05 kernel at 1024^3 (fp16 and tf32 encodings)
OUT=gpurun_out/${1:-ps}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k7_tf32x3 -s 2 -c 1 -o $OUT/k8_1024 \
  python scripts/profile_one.py --variant parallel_fp16x3 --n 1024 --reps 4 > $OUT/k8.log 2>&1; echo "k8 rc=$?" >> $OUT/summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k7_tf32x3 -s 2 -c 1 -o $OUT/k7_1024 \
  python scripts/profile_one.py --variant parallel_tf32x3 --n 1024 --reps 4 > $OUT/k7.log 2>&1; echo "k7 rc=$?" >> $OUT/summary.txt
