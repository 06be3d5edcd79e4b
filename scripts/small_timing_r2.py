"""Small-problem call timing (tuning): per single call with L2 flushed, and
back to back (100 calls event-timed), for the tensor-core encodings and K6."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for n in (1024, 2048):
    for v in ("parallel", "parallel_tf32x3", "parallel_fp16x3"):
        tf = v != "parallel"
        term = schedules.apply("parallel", n, n, n).term
        p = dispatch.decode(term, [(n, n), (n, n)], tf32x3=tf, tc_encoding="fp16" if v.endswith("fp16x3") else "tf32")
        A = torch.empty((n, n), device=dev); synth.fill_device(A, 0, 0)
        B = torch.empty((n, n), device=dev); synth.fill_device(B, 0, 1)
        C = torch.empty((n, n), device=dev)
        call = interp.GemmCall(p, A, B, C, stream)
        for _ in range(5):
            call()
        torch.cuda.synchronize()
        single = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream); call(); e1.record(stream); torch.cuda.synchronize()
            single.append(e0.elapsed_time(e1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(100):
            call()
        e1.record(stream); torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) / 100
        print(json.dumps({"n": n, "variant": v, "fixup": os.environ.get("ELV_TC_FIXUP", "1"),
                          "single_us": 1e3 * statistics.median(single), "b2b_us": 1e3 * b2b,
                          "single_tflops": 2 * n ** 3 / (statistics.median(single) * 1e-3) / 1e12,
                          "b2b_tflops": 2 * n ** 3 / (b2b * 1e-3) / 1e12}), flush=True)
