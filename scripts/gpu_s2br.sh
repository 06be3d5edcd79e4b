#!/bin/bash
OUT=gpurun_out/${1:-s2bs}
mkdir -p $OUT
for rep in 1 2; do
for lib in libelevate_b200.so libelevate_b200_sm32x3.so libelevate_b200_sm32x2.so libelevate_b200_sm8x6.so; do
  for n in 1024 2048 4096; do
  ELV_LIB=$PWD/paper_2002_02268_b200/$lib ONLY_SIMT=1 timeout 300 python scripts/small_timing.py $n $n $n | sed "s/^{/{\"lib\": \"$lib\", /" >> $OUT/small.jsonl 2>> $OUT/small.err
  done
done
done
