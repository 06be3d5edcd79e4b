"""One 3xFP16 call each at 1024^3 (1-CTA kernel) and 3072^3 (pair kernel, by
the pair / 1-CTA model), for an ncu full capture of the two GEMM kernels:
shared-memory (bank) throughput next to the tensor pipe, the evidence for
the shared-memory bound of the narrow 1-CTA tiles."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402

dev = torch.device("cuda", 0)
for n in (1024, 3072):
    p = dispatch.decode(schedules.apply("parallel", n, n, n).term, [(n, n), (n, n)], tf32x3=True, tc_encoding="fp16")
    A = torch.empty((n, n), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((n, n), device=dev); synth.fill_device(B, 0, 1)
    C = torch.empty((n, n), device=dev)
    call = interp.GemmCall(p, A, B, C)
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    print(n, "pair" if interp.pair_kernel(n, n) else "1-CTA", flush=True)
