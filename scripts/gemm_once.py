"""One bench-shape tensor-core GEMM on prepared planes (for ncu captures and
A/B timing): ENC=fp16|tf32, N/K sizes from the env, REPS launches, prints
the median kernel time."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_02268_b200 import _lib, synth  # noqa: E402

M = N = int(os.environ.get("N", 32768))
K = int(os.environ.get("K", 8192))
f16 = os.environ.get("ENC", "fp16") == "fp16"
reps = int(os.environ.get("REPS", 5))
lib = _lib.load()
dev = torch.device("cuda", 0)
A = torch.empty((M, K), device=dev); B = torch.empty((K, N), device=dev)
synth.fill_device(A, 0, 0); synth.fill_device(B, 0, 1)
pre = "elv_fp16x3_" if f16 else "elv_tf32x3_"
ap = torch.empty(getattr(lib, pre + "a_planes_bytes")(M, K), dtype=torch.uint8, device=dev)
bp = torch.empty(getattr(lib, pre + "b_planes_bytes")(N, K), dtype=torch.uint8, device=dev)
C = torch.empty((M, N), device=dev)
st = torch.cuda.current_stream().cuda_stream
_lib.check(getattr(lib, pre + "split_a")(A.data_ptr(), M, K, K, ap.data_ptr(), st), "a")
_lib.check(getattr(lib, pre + "split_b")(B.data_ptr(), K, N, N, bp.data_ptr(), st), "b")
times = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(getattr(lib, pre + "gemm_planes")(ap.data_ptr(), bp.data_ptr(), C.data_ptr(), M, N, K, N, st), "g")
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = statistics.median(times)
out = {"enc": "fp16" if f16 else "tf32", "M": M, "N": N, "K": K, "l2_hints": os.environ.get("ELV_L2_HINTS", "0"),
       "serpentine": os.environ.get("ELV_SERPENTINE", "0"), "ms": ms, "TF": 2.0 * M * N * K / ms / 1e9,
       "times": times}
if os.environ.get("SAVE_C"):          # a sample of C rows for comparing k orders (every 97th row)
    torch.save(C[::97].cpu(), os.environ["SAVE_C"])
print(json.dumps(out), flush=True)
