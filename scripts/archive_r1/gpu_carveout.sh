#!/bin/bash
# A/B of ELV_PREP_CARVEOUT (max-shared carveout on the preparation kernels),
# interleaved, separate processes (the setting is read once per process).
OUT=gpurun_out/${1:-carve}; mkdir -p $OUT
for rep in 1 2; do
for c in 0 1; do
  ELV_PREP_CARVEOUT=$c timeout 300 python scripts/small_timing.py 1024 1024 1024 | sed "s/^{/{\"carveout\": $c, /" >> $OUT/small.jsonl 2>>$OUT/err.log
  ELV_PREP_CARVEOUT=$c timeout 300 python scripts/small_timing.py 2048 2048 2048 | sed "s/^{/{\"carveout\": $c, /" >> $OUT/small.jsonl 2>>$OUT/err.log
  ELV_PREP_CARVEOUT=$c timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline | sed "s/^{/{\"carveout\": $c, /" >> $OUT/bench.jsonl 2>>$OUT/err.log
done
done
echo done >> $OUT/summary.txt
