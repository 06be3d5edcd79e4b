"""Time one kernel variant (prepare + compute separately) and check a row sample.

    ELV_SGEMM_CFG=2 python scripts/time_variant.py --variant parallel --n 8192
"""
import argparse, json, os, statistics, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker only)
from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="parallel")
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--M", type=int, default=0); ap.add_argument("--N", type=int, default=0); ap.add_argument("--K", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
M, N, K = a.M or a.n, a.N or a.n, a.K or a.n
sched, tf = ("parallel", True) if a.variant == "parallel_tf32x3" else (a.variant, False)
dev = torch.device("cuda", 0)
p = dispatch.decode(schedules.apply_padded(sched, M, N, K).term, [(M, K), (K, N)], tf32x3=tf)
A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)
C = torch.empty((M, N), device=dev)
call = interp.GemmCall(p, A, B, C)
for _ in range(3): call()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
comp = []
for _ in range(a.reps):
    flush.zero_()
    call.prepare()
    e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e1.record(); call.compute(); e2.record(); torch.cuda.synchronize()
    comp.append(e1.elapsed_time(e2))
rows = torch.tensor([0, 1, 127, M // 2, M - 1], device=dev)
As, Bh = A[rows].cpu().numpy(), B.cpu().numpy()
ok, worst = oracle.check(C[rows].cpu().numpy(), oracle.mm_f64(As, Bh), oracle.absprod_np(As, Bh), K)
ms = statistics.median(comp)
print(json.dumps({"variant": a.variant, "cfg": os.environ.get("ELV_SGEMM_CFG"), "M": M, "N": N, "K": K,
                  "kernel_ms": ms, "tflops": 2.0 * M * N * K / ms / 1e9, "ok": ok, "worst": worst}), flush=True)
