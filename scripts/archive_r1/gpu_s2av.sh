#!/bin/bash
# A/B: epilogue reading the whole accumulator slice before storing (spills) vs chunk-by-chunk TMA stores
OUT=gpurun_out/${1:-s2av}
mkdir -p $OUT
for i in 1 2 3; do
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/chunk_$i.json 2> $OUT/chunk_$i.err
  ELV_LIB=$PWD/paper_2002_02268_b200/libelevate_b200_readall.so timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/readall_$i.json 2> $OUT/readall_$i.err
done
