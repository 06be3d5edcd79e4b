#!/bin/bash
OUT=gpurun_out/${1:-s2bw}
mkdir -p $OUT
for rep in 1 2; do
  timeout 300 python scripts/small_timing.py 1024 1024 1024 | sed "s/^{/{\"interp\": \"new\", /" >> $OUT/small.jsonl 2>> $OUT/small.err
  cp paper_2002_02268_b200/interp.py /tmp/interp_new.py; cp scripts/_tmp/interp_old.py paper_2002_02268_b200/interp.py
  timeout 300 python scripts/small_timing.py 1024 1024 1024 | sed "s/^{/{\"interp\": \"old\", /" >> $OUT/small.jsonl 2>> $OUT/small.err
  cp /tmp/interp_new.py paper_2002_02268_b200/interp.py
done
