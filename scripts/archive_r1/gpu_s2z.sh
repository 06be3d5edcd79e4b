#!/bin/bash
OUT=gpurun_out/${1:-s2z}
mkdir -p $OUT
for nd in 1 2 3 4; do
  ELV_HOST_D2H_STREAMS=$nd timeout 300 python scripts/host_pipe_trace.py > $OUT/trace_nd$nd.json 2>&1
done
ELV_HOST_D2H_STREAMS=2 timeout 600 python scripts/host_pipe_sweep.py > $OUT/sweep_nd2.jsonl 2>&1
