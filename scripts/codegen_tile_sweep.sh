#!/bin/bash
OUT=gpurun_out/${1:-r2_cg2}; mkdir -p $OUT
for tile in 4x4 8x4 4x8 8x8 2x8; do
  for u in 0 4; do
    ELV_CG_TILE=$tile ELV_CG_UNROLL=$u timeout 300 python scripts/codegen_timing.py 2>>$OUT/err.log | head -1 | sed "s/^{/{\"tile\": \"$tile\", \"unroll\": $u, /" >> $OUT/t.jsonl
  done
done
