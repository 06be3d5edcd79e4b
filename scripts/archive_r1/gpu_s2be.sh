#!/bin/bash
OUT=gpurun_out/${1:-s2be}
mkdir -p $OUT
CONFIGS=grid:-,grow:1024:4096,grow:1024:4096:4096,grow:1024:4096:1024,grow:512:4096,grow:1024:8192,grow:512:8192,grow:1024:2048:4096,grow:2048:4096,grow:256:4096 \
  timeout 1200 python scripts/host_plan_sweep.py > $OUT/sweep.jsonl 2> $OUT/sweep.err
ELV_HOST_PLAN=grow ELV_HOST_STRIPS=1024,4096 timeout 300 python scripts/host_pipe_trace.py > $OUT/trace_1024_4096.json 2> $OUT/trace.err
