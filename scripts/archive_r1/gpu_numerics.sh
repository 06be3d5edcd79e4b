#!/bin/bash
OUT=gpurun_out/${1:-num}
mkdir -p $OUT
for m in 0 1 2 3; do ELV_TF32X3_MODE=$m timeout 300 python scripts/tf32x3_numerics.py > $OUT/mode$m.jsonl 2> $OUT/mode$m.err; done
for m in 0 2; do ELV_TF32X3_MODE=$m timeout 300 python bench.py --workload ladder > $OUT/ladder_mode$m.jsonl 2>&1; done
