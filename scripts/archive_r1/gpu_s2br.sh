#!/bin/bash
OUT=gpurun_out/${1:-s2cb}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp16x3" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
for rep in 1 2; do
for f in 1 0; do
  for n in 1024 2048; do
  ELV_FP16X3_WARP_ROWS=$f timeout 300 python scripts/small_timing.py $n $n $n | grep '"enc": "fp16"' | sed "s/^{/{\"warp_rows\": $f, /" >> $OUT/small.jsonl 2>> $OUT/small.err
  done
done
done
