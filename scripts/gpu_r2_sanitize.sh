#!/bin/bash
# compute-sanitizer over every kernel path (small shapes), round 2: chunked tcgen05 kernels
# (1-CTA and, forced with ELV_TF32X3_PAIR=32, the cta_group::2 kernel), range-guard fix-up,
# pipelined C-ABI row shard; session 4: K7F fused split (pair pass), the narrow small-problem pairs
# (ELV_SMALL_PAIR=64) and the codegen shared-memory tile mode; session 6: the pair
# kernel with the serpentine k order (ELV_SERPENTINE=1)
OUT=gpurun_out/${1:-r2_san}; mkdir -p $OUT
S=$OUT/summary.txt
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?" >> $S
ELV_TF32X3_PAIR=32 timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py --quick > $OUT/memcheck_pair.log 2>&1; echo "memcheck pair rc=$?" >> $S
ELV_TF32X3_PAIR=32 ELV_SERPENTINE=1 timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py --quick > $OUT/memcheck_pair_serpentine.log 2>&1; echo "memcheck pair serpentine rc=$?" >> $S
ELV_SMALL_PAIR=64 timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py --quick > $OUT/memcheck_narrow_pair.log 2>&1; echo "memcheck narrow pair rc=$?" >> $S
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python scripts/sanitize_run.py --quick > $OUT/racecheck.log 2>&1; echo "racecheck rc=$?" >> $S
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize_run.py --quick > $OUT/synccheck.log 2>&1; echo "synccheck rc=$?" >> $S
for t in memcheck memcheck_pair memcheck_pair_serpentine memcheck_narrow_pair racecheck synccheck; do tail -n 2 $OUT/$t.log >> $S; done
