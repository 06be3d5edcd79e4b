#!/bin/bash
OUT=gpurun_out/${1:-s2bo}
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
timeout 1200 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $OUT/summary.txt
