#!/bin/bash
OUT=gpurun_out/${1:-tests}
mkdir -p $OUT
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/summary.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
tail -15 $OUT/pytest_gpu.log >> $OUT/summary.txt
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $OUT/summary.txt
