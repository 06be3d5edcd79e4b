#!/bin/bash
# codegen shared-memory tile mode: outputs per thread x staged iterations, 1024^3 (tuning)
for tile in 4x4 8x4 4x8 8x8; do for tl in 32 64; do
  ELV_CG_SMEM_TILE=$tile ELV_CG_SMEM_TL=$tl python scripts/codegen_timing.py 2>&1 | grep -E '"user|"parallel"' | \
    python -c "import sys,json; [print(json.dumps({'tile':'$tile','tl':$tl,'schedule':d['schedule'],'gflops':round(d['generated_gflops']),'diff':d['max_abs_diff']})) for d in map(json.loads, sys.stdin)]"
done; done
