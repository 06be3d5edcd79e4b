#!/bin/bash
# Serpentine k order of odd waves in the pair kernel (ELV_SERPENTINE=1) against
# the default: interleaved timing at the bench shape, ncu DRAM bytes of one
# launch, and the serpentine result against the default (sampled rows) and
# against the f64 oracle bound.
OUT=gpurun_out/${1:-serpentine}; mkdir -p $OUT
for rep in 1 2 3; do
  for sp in 0 1; do
    for enc in fp16 tf32; do
      ELV_SERPENTINE=$sp ENC=$enc REPS=5 timeout 300 python scripts/gemm_once.py >> $OUT/ab.jsonl 2>> $OUT/err.log
    done
  done
done
for sp in 0 1; do
  for enc in fp16 tf32; do
    ELV_SERPENTINE=$sp ENC=$enc REPS=1 SAVE_C=/tmp/serp_c_${enc}_s$sp.pt timeout 300 python scripts/gemm_once.py >> $OUT/save.jsonl 2>> $OUT/err.log
    ELV_SERPENTINE=$sp ENC=$enc REPS=2 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:k7_tf32x3_pair --launch-skip 1 --launch-count 1 --csv \
      python scripts/gemm_once.py > $OUT/ncu_${enc}_s$sp.csv 2>> $OUT/err.log
  done
done
timeout 600 python scripts/serpentine_check.py /tmp >> $OUT/check.jsonl 2>> $OUT/err.log
rm -f /tmp/serp_c_*.pt
