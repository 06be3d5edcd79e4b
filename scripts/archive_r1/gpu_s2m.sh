#!/bin/bash
OUT=gpurun_out/${1:-s2m}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -n 4 $OUT/pytest_gpu.log >> $S
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
timeout 900 python bench.py --variant parallel --steps 3 --no-cpu-baseline > $OUT/bench_simt.json 2> $OUT/bench_simt.err; echo "bench simt rc=$?" >> $S
