#!/bin/bash
# A/B: fp16 1-CTA N=64 kernel with BK=32 (8 stages) vs BK=64 (4 stages), interleaved
OUT=gpurun_out/${1:-bk}; mkdir -p $OUT
for rep in 1 2; do for bk in 64 32; do
  ELV_FP16_BK64_SMALL=$bk timeout 300 python scripts/fp16_prep_timing.py 2>>$OUT/err.log | grep '"warp_rows": 2, "colmax_slab": "adaptive"' | sed "s/^{/{\"bk\": $bk, /" >> $OUT/t.jsonl
done; done
ELV_FP16_BK64_SMALL=32 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fp16" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
