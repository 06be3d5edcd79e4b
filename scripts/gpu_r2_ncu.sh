#!/bin/bash
# Round-2 ncu evidence: launch list of the bench command + one full capture of the dominant kernel (fp16 pair) and the tf32 pair
OUT=gpurun_out/${1:-r2_ncu}; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ladder > $OUT/launches_bench.log 2>&1; echo "launches rc=$?" >> $OUT/summary.txt
for enc in fp16 tf32; do
  ENC=$enc REPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k7_tf32x3_pair \
    --launch-skip 1 --launch-count 1 -o $OUT/k7_pair_$enc -f python scripts/gemm_once.py > $OUT/ncu_full_$enc.log 2>&1
  echo "full $enc rc=$?" >> $OUT/summary.txt
done
