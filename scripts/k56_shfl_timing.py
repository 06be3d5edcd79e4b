"""cacheBlocks (K5, k56_packed_8x8) timing and a digest of C, for comparing
the LDS.128-fragment build with the warp-shuffle build (ELV_LIB=...k56shfl.so,
compiled with -DELV_K56_SHFL=1).  Tuning evidence."""
import hashlib
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402

dev = torch.device("cuda", 0)
for n in (1024, 4096, 8192):
    p = dispatch.decode(schedules.apply("cacheBlocks", n, n, n).term, [(n, n), (n, n)])
    A = torch.empty((n, n), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((n, n), device=dev); synth.fill_device(B, 0, 1)
    C = torch.empty((n, n), device=dev)
    call = interp.GemmCall(p, A, B, C)
    for _ in range(3):
        call()
    ts = []
    for _ in range(10 if n < 8192 else 5):
        call.prepare()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); call.compute(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    digest = hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"lib": os.path.basename(os.environ.get("ELV_LIB", "libelevate_b200.so")), "n": n,
                      "kernel_ms": round(ms, 4), "tflops": round(2 * n ** 3 / ms / 1e9, 2), "C_sha256": digest}),
          flush=True)
