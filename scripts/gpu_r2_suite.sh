#!/bin/bash
# Round 2: full GPU suite + smoke
OUT=gpurun_out/${1:-r2_suite}; mkdir -p $OUT
S=$OUT/summary.txt
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -3 $OUT/pytest_gpu.log >> $S
