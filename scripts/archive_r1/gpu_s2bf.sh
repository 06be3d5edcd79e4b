#!/bin/bash
OUT=gpurun_out/${1:-s2bf}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rowshard.py -q -p no:cacheprovider > $OUT/pytest_rowshard.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
CONFIGS=grid:-,grow:-,grid:-,grow:- timeout 1200 python scripts/host_plan_sweep.py > $OUT/sweep.jsonl 2> $OUT/sweep.err
SHAPE=16384,16384,8192 CONFIGS=grid:-,grow:- timeout 600 python scripts/host_plan_sweep.py >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
timeout 300 python scripts/host_pipe_trace.py > $OUT/trace_grow.json 2> $OUT/trace.err
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/summary.txt
