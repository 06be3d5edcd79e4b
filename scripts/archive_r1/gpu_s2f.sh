#!/bin/bash
OUT=gpurun_out/${1:-s2f}
mkdir -p $OUT
timeout 300 python scripts/k7_prof.py > $OUT/k7prof_bk32.jsonl 2>&1
ELV_TF32X3_PAIR=16 timeout 300 python scripts/k7_prof.py > $OUT/k7prof_bk16.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "tf32 or parallel or rowshard or smoke" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/summary.txt
