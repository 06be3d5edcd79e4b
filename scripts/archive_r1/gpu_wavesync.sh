#!/bin/bash
OUT=gpurun_out/${1:-ws}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "tf32x3" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $S
tail -2 $OUT/pytest.log >> $S
for r in 1 2 3; do for w in 0 1; do
  echo "== wave_sync=$w rep $r" >> $S
  ELV_WAVE_SYNC=$w timeout 300 python scripts/time_variant.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 3 >> $S 2>>$OUT/err.txt
done; done
for w in 0 1; do
  echo "== ncu wave_sync=$w" >> $S
  ELV_WAVE_SYNC=$w timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:k7_tf32x3 -c 1 \
     python scripts/profile_one.py --variant parallel_tf32x3 --M 32768 --N 32768 --K 8192 --reps 1 2>&1 | grep -E "dram__bytes_read|gpu__time|hit_rate" >> $S
done
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
