"""The cta_group::2 tensor-core kernel alone (mid-size ragged shape, both
encodings, guarded row), for `compute-sanitizer --tool racecheck
--racecheck-report analysis`: its aggregated report names every racing
access pair (sanitizers)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import interp, schedules, synth  # noqa: E402

M, N, K = 1100, 2100, 600
assert interp.pair_kernel(M, N)
A = torch.from_numpy(synth.matrix(M, K, 6, 0)).cuda()
B = torch.from_numpy(synth.matrix(K, N, 6, 1)).cuda()
A[1099, 5] = 2.0 ** -110
for enc in ("tf32", "fp16"):
    C = interp.run_tensor(schedules.apply_padded("parallel", M, N, K).term, A, B, tf32x3=True, tc_encoding=enc)
    torch.cuda.synchronize()
    print(enc, float(C.abs().sum()), flush=True)
