#!/bin/bash
OUT=gpurun_out/${1:-s2n}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "cacheBlocks or codegen" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $S
tail -n 2 $OUT/pytest.log >> $S
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
timeout 900 python scripts/codegen_timing.py > $OUT/codegen_timing.jsonl 2>&1; echo "codegen rc=$?" >> $S
