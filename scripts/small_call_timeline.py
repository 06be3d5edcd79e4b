"""Timeline of one small-problem call (L2 flushed before it): the start / end
of every activity (memset, prepare kernels, GEMM) from the CUDA profiler
(CUPTI via torch.profiler), relative to the first one, per encoding.  Shows
where a 1024^3 call's time goes between launches.  N from the env."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402

n = int(os.environ.get("N", 1024))
dev = torch.device("cuda", 0)
A = torch.empty((n, n), device=dev); synth.fill_device(A, 0, 0)
B = torch.empty((n, n), device=dev); synth.fill_device(B, 0, 1)
C = torch.empty((n, n), device=dev)
flush = torch.empty(64 << 20, device=dev)
term = schedules.apply("parallel", n, n, n).term
for label, tf, enc in (("fp16", True, "fp16"), ("tf32", True, "tf32"), ("simt", False, "tf32")):
    p = dispatch.decode(term, [(n, n), (n, n)], tf32x3=tf, tc_encoding=enc)
    call = interp.GemmCall(p, A, B, C)
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    for rep in range(3):
        flush.fill_(float(rep))
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            call()
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        ev.sort(key=lambda e: e.time_range.start)
        t0 = ev[0].time_range.start if ev else 0
        rows = [{"name": e.name[:60], "start_us": e.time_range.start - t0, "end_us": e.time_range.end - t0}
                for e in ev]
        print(json.dumps({"enc": label, "n": n, "rep": rep, "span_us": (rows[-1]["end_us"] if rows else 0),
                          "activities": rows}), flush=True)
