"""Parallel schedule (SIMT K6, k6_sgemm_ffma2) timing and a digest of C; run
twice, with ELV_K6_BULK=1 selecting the TMA bulk-copy staging variant
(k6_sgemm_bulk).  Tuning evidence."""
import hashlib
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402

dev = torch.device("cuda", 0)
for (M, N, K) in ((4096, 4096, 4096), (8192, 8192, 8192), (32768, 32768, 8192)):
    p = dispatch.decode(schedules.apply("parallel", M, N, K).term, [(M, K), (K, N)])
    A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)
    C = torch.empty((M, N), device=dev)
    call = interp.GemmCall(p, A, B, C)
    for _ in range(2):
        call()
    ts = []
    for _ in range(5 if M < 32768 else 3):
        call.prepare()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); call.compute(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    digest = hashlib.sha256(C[:2048].cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"bulk": os.environ.get("ELV_K6_BULK", "0"), "M": M, "N": N, "K": K, "kernel_ms": round(ms, 3),
                      "tflops": round(2 * M * N * K / ms / 1e9, 2), "C_rows0_2047_sha256": digest}), flush=True)
    del A, B, C, call
    torch.cuda.empty_cache()
