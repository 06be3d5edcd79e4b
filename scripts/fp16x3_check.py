"""Numerics of the 3xFP16 encoding (variant 8) vs 3xTF32 (variant 7) against
the f64 oracle: sampled rows, err/bound (tau from oracle.default_tau), on
U(-1,1) inputs and on inputs with rows/columns scaled over 2^-40..2^40 and a
wide in-row dynamic range."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker)
from paper_2002_02268_b200 import interp, schedules, synth  # noqa: E402


def run_case(M, N, K, kind, enc, dev):
    A = torch.empty((M, K), device=dev); B = torch.empty((K, N), device=dev)
    synth.fill_device(A, 3, 0); synth.fill_device(B, 3, 1)
    if kind == "scaled":
        g = torch.Generator(device="cpu").manual_seed(1)
        rs = torch.pow(2.0, torch.randint(-40, 41, (M, 1), generator=g).float()).to(dev)
        cs = torch.pow(2.0, torch.randint(-40, 41, (1, N), generator=g).float()).to(dev)
        A *= rs
        B *= cs
    elif kind == "dynamic":
        g = torch.Generator(device="cpu").manual_seed(2)
        A *= torch.pow(2.0, torch.randint(-20, 21, (M, K), generator=g).float()).to(dev)
        B *= torch.pow(2.0, torch.randint(-20, 21, (K, N), generator=g).float()).to(dev)
    term = schedules.apply_padded("parallel", M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=enc != "simt", tc_encoding="tf32" if enc == "simt" else enc)
    torch.cuda.synchronize()
    rows = np.r_[0:3, M // 2, M - 2:M]
    Ah, Bh = A[torch.from_numpy(rows).to(dev)].double().cpu().numpy(), B.double().cpu().numpy()
    ref, ab = oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh)
    bnd = oracle.bound(K, ab)
    err = np.abs(C[torch.from_numpy(rows).to(dev)].cpu().numpy().astype(np.float64) - ref)
    r = err / np.maximum(bnd, 1e-300)
    # the deterministic (worst-case) fp32 bound: gamma_K = K u / (1 - K u), u = 2^-24
    u = 2.0 ** -24
    rd = err / np.maximum(K * u / (1 - K * u) * ab, 1e-300)
    return {"M": M, "N": N, "K": K, "inputs": kind, "encoding": enc, "worst": float(r.max()),
            "mean": float(r.mean()), "worst_vs_gammaK": float(rd.max()),
            "finite": bool(np.isfinite(C.cpu().numpy()).all())}


def main():
    dev = torch.device("cuda", 0)
    for (M, N, K) in [(4096, 4096, 512), (4096, 4096, 1024), (4096, 8192, 8192), (8192, 8192, 4096)]:
        for kind in ("uniform", "scaled", "dynamic"):
            for enc in ("tf32", "fp16", "simt"):
                print(json.dumps(run_case(M, N, K, kind, enc, dev)), flush=True)


if __name__ == "__main__":
    main()
