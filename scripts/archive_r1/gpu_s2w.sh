#!/bin/bash
# A/B: sleepy epilogue wait vs plain polling, alternating, same box
OUT=gpurun_out/${1:-s2w}
mkdir -p $OUT
for i in 1 2 3; do
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/sleep_$i.json 2>/dev/null
  ELV_LIB=$PWD/paper_2002_02268_b200/libelevate_b200_nosleep.so timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/poll_$i.json 2>/dev/null
done
