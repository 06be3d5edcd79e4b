#!/bin/bash
OUT=gpurun_out/${1:-bf}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_binomial.py -m gpu -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
for i in 1 2; do timeout 600 python bench.py --workload binomial >> $OUT/bench_bf.jsonl 2>> $OUT/bench_bf.err; done; echo "bench rc=$?" >> $OUT/summary.txt
