#!/bin/bash
OUT=gpurun_out/${1:-s2o}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 900 python -m pytest tests/test_gpu_codegen.py -q --timeout 600 -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $S
tail -n 2 $OUT/pytest.log >> $S
timeout 900 python scripts/codegen_timing.py > $OUT/codegen_timing.jsonl 2>&1; echo "codegen rc=$?" >> $S
