#!/bin/bash
# PDL zeroing kernel instead of the prepare memset: GPU suite on the new
# binary, then the small-shape ladder interleaved against the previous
# binary (ELV_LIB=scripts/_ab/libelevate_b200_before.so), then the bench.
OUT=gpurun_out/${1:-zero_pdl}; mkdir -p $OUT
S=$OUT/summary.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -2 $OUT/pytest_gpu.log >> $S
for rep in 1 2; do
  ELV_LIB=$PWD/scripts/_ab/libelevate_b200_before.so timeout 600 python scripts/ladder_small.py > $OUT/ladder_before_$rep.jsonl 2>> $OUT/err.log
  timeout 600 python scripts/ladder_small.py > $OUT/ladder_after_$rep.jsonl 2>> $OUT/err.log
done
timeout 900 python bench.py --no-ladder > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
