"""Run one kernel variant a few times (for ncu captures).

    ncu --set full --clock-control none --import-source on -k regex:k7_tf32x3 -s 2 -c 1 \
        -o gpurun_out/prof python scripts/profile_one.py --variant parallel_tf32x3 --n 8192
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="parallel_tf32x3")
    ap.add_argument("--M", type=int, default=0)
    ap.add_argument("--N", type=int, default=0)
    ap.add_argument("--K", type=int, default=0)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    M, N, K = a.M or a.n, a.N or a.n, a.K or a.n
    sched, tf = ("parallel", True) if a.variant.startswith("parallel_") else (a.variant, False)
    enc = "fp16" if a.variant == "parallel_fp16x3" else "tf32"
    dev = torch.device("cuda", 0)
    term = schedules.apply_padded(sched, M, N, K).term
    p = dispatch.decode(term, [(M, K), (K, N)], tf32x3=tf, tc_encoding=enc)
    A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)
    C = torch.empty((M, N), device=dev)
    call = interp.GemmCall(p, A, B, C)
    for _ in range(a.reps):
        call()
    torch.cuda.synchronize()
    print("ok", a.variant, M, N, K)


if __name__ == "__main__":
    main()
