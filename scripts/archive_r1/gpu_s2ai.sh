#!/bin/bash
# power/rate experiment: kind::f16 MMAs on the same operand bytes (wrong results)
OUT=gpurun_out/${1:-s2ai}
mkdir -p $OUT
for i in 1 2; do
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/tf32_$i.json 2>/dev/null
  ELV_LIB=$PWD/paper_2002_02268_b200/libelevate_b200_f16x.so timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/f16_$i.json 2>/dev/null
done
