#!/bin/bash
# Session-6 final evidence on the current binary: session-end set (smoke, GPU
# suite, bench, ladder, launch list) + one ncu --set full capture of the
# bench-shape dominant kernel (3xFP16 pair).
TAG=${1:-s6final}
bash scripts/gpu_session_end.sh $TAG
OUT=gpurun_out/$TAG
ENC=fp16 REPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k7_tf32x3_pair \
  --launch-skip 1 --launch-count 1 -o $OUT/k7_pair_fp16 -f python scripts/gemm_once.py > $OUT/ncu_full_fp16.log 2>&1
echo "ncu full fp16 rc=$?" >> $OUT/summary.txt
ncu -i $OUT/k7_pair_fp16.ncu-rep --page raw --csv > $OUT/k7_pair_fp16_raw.csv 2>> $OUT/ncu_full_fp16.log
rm -f $OUT/k7_pair_fp16.ncu-rep
