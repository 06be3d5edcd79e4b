"""A few calls per variant at small shapes, for an ncu launch list:
    ncu --metrics gpu__time_duration.sum --csv python scripts/small_launches.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import interp, schedules, synth  # noqa: E402

dev = torch.device("cuda", 0)
for n in (1024, 2048, 4096):
    A = torch.empty((n, n), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((n, n), device=dev); synth.fill_device(B, 0, 1)
    for tf, enc in ((True, "tf32"), (True, "fp16")):
        p = interp.plan(schedules.apply("parallel", n, n, n).term, [(n, n), (n, n)], tf, enc)
        call = interp.GemmCall(p, A, B, torch.empty((n, n), device=dev))
        for _ in range(2):
            call()
        torch.cuda.synchronize()
        print("done", n, enc, p.variant, flush=True)
