#!/bin/bash
OUT=gpurun_out/${1:-bf}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_binomial.py -q --timeout 300 -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
tail -15 $OUT/pytest.log >> $OUT/summary.txt
timeout 600 python bench.py --workload binomial > $OUT/bench_bf.jsonl 2> $OUT/bench_bf.err; echo "bench rc=$?" >> $OUT/summary.txt
timeout 600 ncu --set full --clock-control none -k regex:k_bf_band -s 6 -c 2 -o $OUT/prof_bf python bench.py --workload binomial --steps 1 > $OUT/prof.log 2>&1; echo "ncu rc=$?" >> $OUT/summary.txt
