#!/bin/bash
# 1024^3: per-kernel durations (ncu launch list) and single / back-to-back call timing
OUT=gpurun_out/${1:-small_prof}; mkdir -p $OUT
timeout 300 python scripts/small_timing_r2.py > $OUT/small_timing.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file $OUT/launches.csv \
  python scripts/small_call_launches.py > $OUT/launches.log 2>&1
echo done >> $OUT/summary.txt
