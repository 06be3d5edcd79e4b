"""Time 3xTF32 fused (K7F, one launch + fix-up) against the planes path
(split prepass + pair kernel + fix-up) on the same inputs, whole call and
kernel alone, L2 flushed before each rep.  Tuning evidence.

    python scripts/fused_timing.py --shapes 8192,8192,8192 32768,32768,8192
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import _lib, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", nargs="+", default=["8192,8192,8192", "32768,32768,8192"])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dbg", nargs="*", type=int, default=[], help="ELV_K7F_DBG values to time the fused kernel with")
a = ap.parse_args()
lib = _lib.load()
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def ev():
    return torch.cuda.Event(enable_timing=True)


for sh in a.shapes:
    M, N, K = map(int, sh.split(","))
    A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)
    C = torch.empty((M, N), device=dev)
    st = torch.cuda.current_stream().cuda_stream
    ap_ = torch.empty(lib.elv_tf32x3_a_planes_bytes(M, K), dtype=torch.uint8, device=dev)
    bp_ = torch.empty(lib.elv_tf32x3_b_planes_bytes(N, K), dtype=torch.uint8, device=dev)
    flags = torch.empty(M + N, dtype=torch.int32, device=dev)

    def fused():
        _lib.check(lib.elv_tf32x3_gemm_fused(A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, M, N, K,
                                             flags.data_ptr(), st), "fused")

    def split():
        _lib.check(lib.elv_tf32x3_split_a(A.data_ptr(), M, K, K, ap_.data_ptr(), st), "sa")
        _lib.check(lib.elv_tf32x3_split_b(B.data_ptr(), K, N, N, bp_.data_ptr(), st), "sb")

    def planes_gemm():
        _lib.check(lib.elv_tf32x3_gemm_planes(ap_.data_ptr(), bp_.data_ptr(), C.data_ptr(), M, N, K, N, st), "g")
        _lib.check(lib.elv_tc_fixup(7, ap_.data_ptr(), bp_.data_ptr(), A.data_ptr(), K, B.data_ptr(), N, 0,
                                    C.data_ptr(), N, M, N, K, st), "fix")

    def split_b():
        _lib.check(lib.elv_tf32x3_split_b(B.data_ptr(), K, N, N, bp_.data_ptr(), st), "sb")

    def fused_a():
        _lib.check(lib.elv_tf32x3_gemm_fused_a(A.data_ptr(), K, bp_.data_ptr(), B.data_ptr(), N, C.data_ptr(), N,
                                               M, N, K, flags.data_ptr(), st), "fused_a")

    res = {"M": M, "N": N, "K": K}
    cases = [("fused", [fused], 0), ("planes", [split, planes_gemm], 0), ("planes_gemm_only", [planes_gemm], 0)]
    cases += [("hybrid", [split_b, fused_a], 0), ("hybrid_gemm_only", [fused_a], 0)]
    cases += [(f"fused_dbg{d}", [fused], d) for d in a.dbg]
    for name, fns, dbg in cases:
        os.environ["ELV_K7F_DBG"] = str(dbg)
        for _ in range(2):
            for f in ([split] if name.endswith("gemm_only") else []) + fns:
                f()
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            if name.endswith("gemm_only"):
                split()
            e1, e2 = ev(), ev()
            e1.record()
            for f in fns:
                f()
            e2.record()
            torch.cuda.synchronize()
            ts.append(e1.elapsed_time(e2))
        ms = statistics.median(ts)
        res[name] = {"ms": round(ms, 4), "tflops": round(2.0 * M * N * K / ms / 1e9, 1)}
    print(json.dumps(res), flush=True)
