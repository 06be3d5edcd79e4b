#!/bin/bash
OUT=gpurun_out/${1:-cp}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowshard.py -q --timeout 300 -k "parallel and not tf32x3" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $OUT/pytest.log >> $S
for r in 1 2; do for c in 1 0; do
  ELV_SGEMM_CP=$c timeout 120 python scripts/time_variant.py --variant parallel --n 8192 >> $S 2>>$OUT/err.txt
  ELV_SGEMM_CP=$c timeout 300 python scripts/time_variant.py --variant parallel --M 32768 --N 32768 --K 8192 --reps 2 >> $S 2>>$OUT/err.txt
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k6_sgemm_cp -s 1 -c 1 -o $OUT/prof_cp \
  python scripts/profile_one.py --variant parallel --n 8192 --reps 2 > $OUT/prof.log 2>&1
