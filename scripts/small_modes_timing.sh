#!/bin/bash
# 1024^3 single-call timing of the small-problem paths: fused fp16 prepare and in-kernel fix-up on/off
for fp in 1 0; do for ik in 1 0; do
  echo "fused_prep=$fp fixup_inkernel=$ik"
  ELV_FP16X3_FUSED_PREP=$fp ELV_TC_FIXUP_INKERNEL=$ik python scripts/small_timing_r2.py 2>&1 | grep '"n": 1024'
done; done
