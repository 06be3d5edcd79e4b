#!/bin/bash
OUT=gpurun_out/${1:-ord}
mkdir -p $OUT
S=$OUT/summary.txt
for r in 1 2; do for o in 2 3; do
  echo "order $o" >> $S
  ELV_SGEMM_ORDER=$o timeout 120 python scripts/time_variant.py --variant parallel --n 8192 >> $S 2>>$OUT/err.txt
done; done
