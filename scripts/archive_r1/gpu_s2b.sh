#!/bin/bash
# host pipeline (elv_gemm_host): tests + bench e2e
OUT=gpurun_out/${1:-s2b}
mkdir -p $OUT
S=$OUT/summary.txt
timeout 900 python -m pytest tests/test_gpu_rowshard.py -q --timeout 600 -p no:cacheprovider > $OUT/pytest_rowshard.log 2>&1; echo "pytest rc=$?" >> $S
tail -4 $OUT/pytest_rowshard.log >> $S
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
timeout 900 python bench.py --no-cpu-baseline --variant parallel --steps 3 > $OUT/bench_simt.json 2> $OUT/bench_simt.err; echo "bench rc=$?" >> $S
