#!/bin/bash
# End-of-session evidence: smoke, full GPU suite, default bench, ladder, launch list.
OUT=gpurun_out/${1:-end}; mkdir -p $OUT
S=$OUT/summary.txt
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -2 $OUT/pytest_gpu.log >> $S
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1; echo "launches rc=$?" >> $S
