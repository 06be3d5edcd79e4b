#!/bin/bash
# power-cap sensitivity: K7 with half the L2->SMEM traffic (hi planes only; wrong results)
OUT=gpurun_out/${1:-s2ad}
mkdir -p $OUT
for i in 1 2; do
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/full_$i.json 2>/dev/null
  ELV_LIB=$PWD/paper_2002_02268_b200/libelevate_b200_nolo.so timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/nolo_$i.json 2>/dev/null
done
