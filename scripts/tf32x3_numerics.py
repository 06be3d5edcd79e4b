"""Diagnostics: error of the tcgen05 3xTF32 kernel vs K, per MMA schedule.

Run on a GPU box:  python scripts/tf32x3_numerics.py  (ELV_TF32X3_LOLO=0/1 forces lo.lo off/on)
Prints, per K: worst and mean err/bound (bound = sqrt(K) 2^-24 |A||B|) and the
mean signed error relative to |A||B| (bias), for the GPU kernel, the SIMT
parallel kernel, and a host model with exact (f64) accumulation of the same
hi/lo products (isolates representation error from accumulation error).
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402


def rna_tf32(x):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return u.view(np.float32)


def stats(C, ref, ab, K):
    b = oracle.bound(K, ab)
    r = np.abs(C - ref) / b
    return {"worst": float(r.max()), "mean": float(r.mean()),
            "bias": float(((C - ref) / ab).mean() * 2 ** 24)}


def main():
    mode = os.environ.get("ELV_TF32X3_LOLO", "auto")
    dev = torch.device("cuda", 0)
    M = N = 256
    rows = []
    for K in (1, 4, 8, 17, 64, 256, 1024, 4096, 8192):
        A = torch.empty((M, K), device=dev); synth.fill_device(A, 4, 0)
        B = torch.empty((K, N), device=dev); synth.fill_device(B, 4, 1)
        Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
        ref = oracle.mm_f64(Ah, Bh)
        ab = oracle.absprod_np(Ah, Bh)
        out = {"K": K, "mode": mode}
        for v, tf in (("tc", True), ("simt", False)):
            term = schedules.apply_padded("parallel", M, N, K).term
            C = interp.run_tensor(term, A, B, tf32x3=tf).cpu().numpy().astype(np.float64)
            out[v] = stats(C, ref, ab, K)
        ah, bh = rna_tf32(Ah), rna_tf32(Bh)
        al, bl = rna_tf32(Ah - ah), rna_tf32(Bh - bh)
        f = lambda x: x.astype(np.float64)
        model3 = f(ah) @ f(bh) + f(ah) @ f(bl) + f(al) @ f(bh)
        model4 = model3 + f(al) @ f(bl)
        out["model3_exact_acc"] = stats(model3, ref, ab, K)
        out["model4_exact_acc"] = stats(model4, ref, ab, K)
        rows.append(out)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
