#!/bin/bash
# compute-sanitizer over every kernel path (small shapes)
OUT=gpurun_out/${1:-s2k}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?" >> $S
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python scripts/sanitize_run.py --quick > $OUT/racecheck.log 2>&1; echo "racecheck rc=$?" >> $S
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize_run.py --quick > $OUT/synccheck.log 2>&1; echo "synccheck rc=$?" >> $S
for t in memcheck racecheck synccheck; do tail -n 2 $OUT/$t.log >> $S; done
