#!/bin/bash
OUT=gpurun_out/${1:-s2bl}
mkdir -p $OUT
for f in 0 1; do
  ELV_K6_SMALL_PDL=$f timeout 300 python scripts/small_timing.py 1024 1024 1024 | sed "s/^{/{\"k6_small_pdl\": $f, /" >> $OUT/small.jsonl 2>> $OUT/small.err
done
for pdl in 1 0; do
  for n in 2048 4096 8192; do
    ELV_PDL=$pdl timeout 300 python scripts/small_timing.py $n $n $n | sed "s/^{/{\"pdl\": $pdl, /" >> $OUT/small.jsonl 2>> $OUT/small.err
  done
done
