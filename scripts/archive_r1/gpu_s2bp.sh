#!/bin/bash
OUT=gpurun_out/${1:-s2bp}
mkdir -p $OUT
for rep in 1 2; do
  for pace in 0 2 4 8 16; do
    ELV_HOST_PACE=$pace CONFIGS=grow:- timeout 600 python scripts/host_plan_sweep.py >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
  done
done
ELV_HOST_PACE=4 timeout 300 python scripts/host_pipe_trace.py > $OUT/trace_pace4.json 2> $OUT/trace.err
