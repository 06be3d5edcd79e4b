#!/bin/bash
OUT=gpurun_out/${1:-s2ca}
mkdir -p $OUT
for rep in 1 2; do
for lib in libelevate_b200.so libelevate_b200_cp64x2.so libelevate_b200_cp48x3.so libelevate_b200_cp40x3.so; do
  ELV_LIB=$PWD/paper_2002_02268_b200/$lib ONLY_SIMT=1 timeout 300 python scripts/small_timing.py 8192 8192 8192 | sed "s/^{/{\"lib\": \"$lib\", /" >> $OUT/small.jsonl 2>> $OUT/small.err
done
done
