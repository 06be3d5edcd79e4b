#!/bin/bash
OUT=gpurun_out/${1:-s2bx}
mkdir -p $OUT
for rep in 1 2; do
for nt in 64 128; do
  for n in 1024 2048 4096; do
  ELV_K6_SMALL_THREADS=$nt ONLY_SIMT=1 timeout 300 python scripts/small_timing.py $n $n $n | sed "s/^{/{\"nt\": $nt, /" >> $OUT/small.jsonl 2>> $OUT/small.err
  done
done
done
ELV_K6_SMALL_THREADS=128 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "parallel or small or odd" -p no:cacheprovider > $OUT/pytest128.log 2>&1; echo "pytest128 rc=$?" >> $OUT/summary.txt
