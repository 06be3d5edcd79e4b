"""What one rank of the 8-GPU row-sharded bench step costs, measured on one
B200, plus the NCCL broadcast the model adds for an assumed bus bandwidth
(no second GPU in this environment: an estimate, not a measurement of
scaling).  Readiness evidence for DESIGN.md section 6.

Runs PipelinedRowShardGemm (the bench's step: packedB in column chunks, split
on arrival, GEMM + fix-up per chunk) in a one-process world on
  * the full problem (32768 rows)            -> T1
  * one rank's shard at 8 ranks (4096 rows)   -> T_rank (incl. rank 0's packing)
and per-chunk GEMM times, then models
  step_8 = T_rank + bcast(chunk 0) + sum_c max(0, bcast(chunk c) - gemm(chunk c-1))
  efficiency = T1 / (8 * step_8)
for NCCL broadcast bus bandwidths of 300 / 450 / 600 GB/s, for each chunk
count in CHUNKS (default 4, the bench's).
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import dispatch, distributed, schedules, synth  # noqa: E402

dev = torch.device("cuda", 0)
N, K = 32768, 8192
B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)


def step_time(M, reps=5, chunks=4):
    term = schedules.apply("parallel", 32768, N, K).term
    plan = dispatch.decode(term, [(M, K), (K, N)], tf32x3=True, tc_encoding="fp16")
    A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
    C = torch.empty((M, N), device=dev)
    pipe = distributed.PipelinedRowShardGemm(plan, N, K, dev, chunks=chunks)
    for _ in range(2):
        pipe.step(A, B, C)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pipe.step(A, B, C); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), pipe.chunks


t1, _ = step_time(32768, reps=3)
for nchunks in [int(c) for c in os.environ.get("CHUNKS", "4").split(",")]:
    tr, chunks = step_time(4096, chunks=nchunks)
    widths = [n1 - n0 for n0, n1 in chunks]
    gemm_c = [tr * w / N for w in widths]                       # per-chunk share of the rank's step
    out = {"T1_ms": t1, "T_rank_ms_4096_rows": tr, "chunks": widths, "model": []}
    for bw in (300, 450, 600):
        b = [((w + 255) // 256) * 256 * K * 4 / (bw * 1e9) * 1e3 for w in widths]   # ms per chunk broadcast
        exposed = b[0] + sum(max(0.0, b[c] - gemm_c[c - 1]) for c in range(1, len(b)))
        step8 = tr + exposed
        out["model"].append({"nccl_broadcast_busbw_GBps": bw, "exposed_broadcast_ms": exposed, "step_8_ms": step8,
                             "efficiency_8": t1 / (8 * step8)})
    print(json.dumps(out), flush=True)
