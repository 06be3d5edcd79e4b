"""Mid-size problems (fewer 256x256 pair tiles than SMs): the tensor-core
GEMM launch (planes prepared, range-guard fix-up included, L2 flushed) and a
digest of C, for the kernel the library picks -- run once with the defaults
and once with ELV_TF32X3_PAIR=32 (forces the cta_group::2 kernel; read once
per process).  Tuning evidence for the pair / 1-CTA crossover (DESIGN.md
section 12)."""
import hashlib
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402

SHAPES = [tuple(int(x) for x in s.split("x")) for s in
          os.environ.get("SHAPES", "1536x1536x1536,2048x2048x2048,2048x4096x2048,2560x2560x2560,"
                                   "3072x3072x3072,2048x2048x8192").split(",")]
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for (M, N, K) in SHAPES:
    A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
    B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)
    for enc in ("fp16", "tf32"):
        p = dispatch.decode(schedules.apply("parallel", M, N, K).term, [(M, K), (K, N)], tf32x3=True,
                            tc_encoding=enc)
        C = torch.empty((M, N), device=dev)
        call = interp.GemmCall(p, A, B, C)
        for _ in range(3):
            call()
        ts, tc = [], []
        for _ in range(15):
            flush.zero_()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(); call.prepare(); e1.record(); call.compute(); e2.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e2)); tc.append(e1.elapsed_time(e2))
        us, cus = 1e3 * statistics.median(ts), 1e3 * statistics.median(tc)
        print(json.dumps({"M": M, "N": N, "K": K, "enc": enc, "pair_forced": os.environ.get("ELV_TF32X3_PAIR", "auto"),
                          "compute_us": round(cus, 2), "call_us": round(us, 2),
                          "compute_tflops": round(2 * M * N * K / cus / 1e6, 1),
                          "C_sha256": hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()[:16]}), flush=True)
    del A, B
