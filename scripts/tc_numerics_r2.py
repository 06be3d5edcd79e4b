"""Round-2 numerics probe of the tensor-core encodings (K7 3xTF32, K8 3xFP16)
against the SIMT kernel and the f64 oracle on adversarial input classes:

  uniform   U(-1,1)
  positive  U(0,1) (no cancellation: |C| = (|A||B|), the accumulator's
            round-toward-zero bias adds up)
  dominant  U(-1,1) with one element per row of A scaled by 2^12
  outlier0  row i of A has A[i,0] = 2^32, and B[0,:] = 0 (the outlier meets zeros)
  huge      rows of A scaled by 2^110, columns of B by 2^-110
  dynamic   every element scaled by 2^u, u uniform in [-20, 20]

worst / mean err / bound(tau) over sampled rows; prints one JSON line per case.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker)
from paper_2002_02268_b200 import interp, schedules, synth  # noqa: E402


def make(M, N, K, kind, dev):
    A = torch.empty((M, K), device=dev); B = torch.empty((K, N), device=dev)
    synth.fill_device(A, 5, 0); synth.fill_device(B, 5, 1)
    g = torch.Generator(device="cpu").manual_seed(7)
    if kind == "positive":
        A.abs_(); B.abs_()
    elif kind == "dominant":
        idx = torch.randint(0, K, (M,), generator=g).to(dev)
        A[torch.arange(M, device=dev), idx] *= 4096.0
    elif kind == "outlier0":
        A[:, 0] = 2.0 ** 32
        B[0, :] = 0.0
    elif kind == "huge":
        A *= 2.0 ** 110
        B *= 2.0 ** -110
    elif kind == "dynamic":
        A *= torch.pow(2.0, torch.randint(-20, 21, (M, K), generator=g).float()).to(dev)
        B *= torch.pow(2.0, torch.randint(-20, 21, (K, N), generator=g).float()).to(dev)
    return A, B


def run_case(M, N, K, kind, enc, dev, A, B):
    term = schedules.apply_padded("parallel", M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=enc != "simt", tc_encoding="tf32" if enc == "simt" else enc)
    torch.cuda.synchronize()
    rows = np.unique(np.r_[0:4, np.linspace(0, M - 1, 28).astype(int)])
    ri = torch.from_numpy(rows).to(dev)
    Ah, Bh = A[ri].double().cpu().numpy(), B.double().cpu().numpy()
    ref, ab = oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh)
    bnd = oracle.bound(K, ab)
    Cr = C[ri].cpu().numpy().astype(np.float64)
    err = np.abs(Cr - ref)
    r = err / np.maximum(bnd, 1e-300)
    return {"M": M, "N": N, "K": K, "inputs": kind, "encoding": enc, "worst": float(np.nanmax(r)),
            "mean": float(np.nanmean(r)), "finite": bool(np.isfinite(Cr).all())}


def main():
    dev = torch.device("cuda", 0)
    shapes = [(2048, 2048, 512), (2048, 2048, 2048), (4096, 4096, 8192)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
    for (M, N, K) in shapes:
        for kind in ("uniform", "positive", "dominant", "outlier0", "huge", "dynamic"):
            A, B = make(M, N, K, kind, dev)
            for enc in ("tf32", "fp16", "simt"):
                print(json.dumps(run_case(M, N, K, kind, enc, dev, A, B)), flush=True)


if __name__ == "__main__":
    main()
