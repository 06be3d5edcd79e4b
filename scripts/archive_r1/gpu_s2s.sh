#!/bin/bash
OUT=gpurun_out/${1:-s2s}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -n 3 $OUT/pytest_gpu.log >> $S
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
ELV_PDL=0 timeout 900 python bench.py --workload ladder > $OUT/ladder_nopdl.jsonl 2> $OUT/ladder_nopdl.err; echo "ladder nopdl rc=$?" >> $S
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py --quick > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?" >> $S
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
