"""Serpentine experiment check (scripts/gpu_serpentine.sh): the sampled C rows
(every 97th) of the default and the serpentine pair kernel at the bench
shape, compared with each other and against the f64 product (computed on
the GPU in float64, test infrastructure only) under the tau = 1 sqrt(K) bound
of oracle.bound."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2002_02268_b200 import synth  # noqa: E402

out = sys.argv[1]
M = N = int(os.environ.get("N", 32768))
K = int(os.environ.get("K", 8192))
dev = torch.device("cuda", 0)
A = torch.empty((M, K), device=dev)
B = torch.empty((K, N), device=dev)
synth.fill_device(A, 0, 0)
synth.fill_device(B, 0, 1)
As = A[::97].double()
Bd = B.double()
ref = (As @ Bd).cpu().numpy()
ab = (As.abs() @ Bd.abs()).cpu().numpy()
del Bd
for enc in ("fp16", "tf32"):
    c0 = torch.load(os.path.join(out, f"serp_c_{enc}_s0.pt")).numpy()
    c1 = torch.load(os.path.join(out, f"serp_c_{enc}_s1.pt")).numpy()
    ok0, w0 = oracle.check(c0, ref, ab, K)
    ok1, w1 = oracle.check(c1, ref, ab, K)
    diff = c0 != c1
    rel = np.abs(c0.astype(np.float64) - c1) / np.maximum(np.abs(c0.astype(np.float64)), 1e-30)
    print(json.dumps({"enc": enc, "rows_sampled": int(c0.shape[0]), "default_ok": ok0, "default_worst": w0,
                      "serpentine_ok": ok1, "serpentine_worst": w1,
                      "frac_elements_differ": float(diff.mean()), "max_rel_diff": float(rel.max())}), flush=True)
