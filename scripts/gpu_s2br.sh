#!/bin/bash
OUT=gpurun_out/${1:-s2bu}
mkdir -p $OUT
for lib in libelevate_b200.so libelevate_b200_k34.so; do
  for n in 1024 8192; do
  ELV_LIB=$PWD/paper_2002_02268_b200/$lib SCHEDS=loopPerm,arrayPacking,cacheBlocks timeout 300 python scripts/small_timing.py $n $n $n | sed "s/^{/{\"lib\": \"$lib\", /" >> $OUT/small.jsonl 2>> $OUT/small.err
  done
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_codegen.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
