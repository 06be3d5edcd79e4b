#!/bin/bash
# ncu full captures of the 1024^3 GEMM kernels (3xFP16 1-CTA, 3xTF32 1-CTA, SIMT k6_sgemm_small)
OUT=gpurun_out/${1:-small_ncu}; mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k7_tf32x3|k6_sgemm_small|k16_prep|k16_split|k_tc_fixup" \
  --launch-skip 0 --launch-count 40 -o $OUT/small -f python scripts/small_call_launches.py > $OUT/ncu.log 2>&1
echo "rc=$?" >> $OUT/summary.txt
