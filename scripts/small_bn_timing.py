"""Time the 3xFP16 / 3xTF32 GEMM launch alone (planes prepared) at a small
shape, for the N tile forced by ELV_TF32X3_BN (read once per process)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402

n = int(os.environ.get("N", 1024))
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for enc in ("fp16", "tf32"):
    term = schedules.apply("parallel", n, n, n).term
    p = dispatch.decode(term, [(n, n), (n, n)], tf32x3=True, tc_encoding=enc)
    A = torch.empty((n, n), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((n, n), device=dev); synth.fill_device(B, 0, 1)
    C = torch.empty((n, n), device=dev)
    call = interp.GemmCall(p, A, B, C)
    for _ in range(3):
        call()
    ts = []
    for _ in range(20):
        call.prepare()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); call.compute(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    us = 1e3 * statistics.median(ts)
    print(json.dumps({"n": n, "enc": enc, "bn": os.environ.get("ELV_TF32X3_BN", "auto"), "compute_us": round(us, 2),
                      "tflops": round(2 * n ** 3 / us / 1e6, 1)}), flush=True)
