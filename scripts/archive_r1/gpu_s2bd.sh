#!/bin/bash
# growing-schedule host pipeline: tests, plan sweep, trace
OUT=gpurun_out/${1:-s2bd}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rowshard.py -q -x -k "host" -p no:cacheprovider > $OUT/pytest_host.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
timeout 900 python scripts/host_plan_sweep.py > $OUT/sweep.jsonl 2> $OUT/sweep.err
SHAPE=16384,16384,8192 timeout 600 python scripts/host_plan_sweep.py >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
SHAPE=8192,8192,8192 CONFIGS=grid:-,grow:- timeout 600 python scripts/host_plan_sweep.py >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
timeout 300 python scripts/host_pipe_trace.py > $OUT/trace_fp16.json 2> $OUT/trace.err
