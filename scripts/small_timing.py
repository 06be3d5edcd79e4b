"""Device time of one interp.run_tensor call (prepare + GEMM) at small
shapes, per variant / encoding, CUDA events, median of 50 after warm-up.

    python scripts/small_timing.py [M N K]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import interp, schedules, synth  # noqa: E402


def main():
    M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (1024, 1024, 1024)
    dev = torch.device("cuda", 0)
    A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)
    cases = [("parallel", False, "tf32"), ("parallel", True, "tf32"), ("parallel", True, "fp16")]
    if os.environ.get("ONLY_SIMT"):
        cases = cases[:1]
    if os.environ.get("SCHEDS"):
        cases = [(x, False, "tf32") for x in os.environ["SCHEDS"].split(",")]
    for sched, tf, enc in cases:
        term = schedules.apply_padded(sched, M, N, K).term
        p = interp.plan(term, [(M, K), (K, N)], tf, enc)
        call = interp.GemmCall(p, A, B, torch.empty((M, N), device=dev))
        for _ in range(10):
            call()
        ts = []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); call(); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        # back to back (launch-rate bound if the host is slower than the GPU)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(200):
            call()
        e1.record()
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) / 200
        # CUDA graph of one call, replayed (no host launch cost)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            gc = interp.GemmCall(p, A, B, call.C, stream=s)
            gc()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                gc()
        torch.cuda.synchronize()
        for _ in range(5):
            g.replay()
        e0.record()
        for _ in range(200):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        gr = e0.elapsed_time(e1) / 200
        print(json.dumps({"shape": [M, N, K], "sched": sched, "variant": p.variant, "enc": enc, "us_single": round(ms * 1e3, 2),
                          "us_back_to_back": round(b2b * 1e3, 2), "us_graph": round(gr * 1e3, 2),
                          "TFLOP/s_single": round(2.0 * M * N * K / ms / 1e9, 1),
                          "TFLOP/s_graph": round(2.0 * M * N * K / gr / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
