#!/bin/bash
# ncu full captures of the fused / hybrid 3xTF32 kernel and the planes pair kernel at 8192^3
OUT=gpurun_out/${1:-fused_ncu}; mkdir -p $OUT
for mode in fused hybrid planes; do
  if [ $mode = planes ]; then K=regex:k7_tf32x3_pair; else K=regex:k7f; fi
  MODE=$mode timeout 600 ncu --set full --import-source on --clock-control none -k $K --launch-skip 1 --launch-count 1 \
    -o $OUT/$mode -f python scripts/fused_once.py > $OUT/$mode.log 2>&1
  echo "$mode rc=$?" >> $OUT/summary.txt
done
