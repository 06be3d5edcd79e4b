"""One elv_gemm call (prepare + compute) per encoding at a small shape, for
ncu launch lists (N, K from the env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_02268_b200 import interp, schedules, synth  # noqa: E402

n = int(os.environ.get("N", 1024))
dev = torch.device("cuda", 0)
A = torch.empty((n, n), device=dev); synth.fill_device(A, 0, 0)
B = torch.empty((n, n), device=dev); synth.fill_device(B, 0, 1)
term = schedules.apply("parallel", n, n, n).term
for enc in ("tf32", "fp16"):
    for _ in range(3):
        interp.run_tensor(term, A, B, tf32x3=True, tc_encoding=enc)
    torch.cuda.synchronize()
for _ in range(3):
    interp.run_tensor(term, A, B, tf32x3=False)
torch.cuda.synchronize()
