"""Run the 3xTF32 fused (K7F), hybrid (A fused, B planes) or planes GEMM a few
times on one shape (for ncu captures of k7f_tf32x3_fused / k7_tf32x3_pair).

    MODE=fused N=8192 ncu --set full -k regex:k7f -s 1 -c 1 -o out python scripts/fused_once.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import _lib, synth  # noqa: E402

mode = os.environ.get("MODE", "fused")
n = int(os.environ.get("N", "8192"))
M = N = K = n
lib = _lib.load()
dev = torch.device("cuda", 0)
A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)
C = torch.empty((M, N), device=dev)
st = torch.cuda.current_stream().cuda_stream
ap_ = torch.empty(lib.elv_tf32x3_a_planes_bytes(M, K), dtype=torch.uint8, device=dev)
bp_ = torch.empty(lib.elv_tf32x3_b_planes_bytes(N, K), dtype=torch.uint8, device=dev)
flags = torch.empty(M + N, dtype=torch.int32, device=dev)
for _ in range(int(os.environ.get("REPS", "2"))):
    if mode == "fused":
        _lib.check(lib.elv_tf32x3_gemm_fused(A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, M, N, K,
                                             flags.data_ptr(), st), "fused")
    elif mode == "hybrid":
        _lib.check(lib.elv_tf32x3_split_b(B.data_ptr(), K, N, N, bp_.data_ptr(), st), "sb")
        _lib.check(lib.elv_tf32x3_gemm_fused_a(A.data_ptr(), K, bp_.data_ptr(), B.data_ptr(), N, C.data_ptr(), N,
                                               M, N, K, flags.data_ptr(), st), "fused_a")
    else:
        _lib.check(lib.elv_tf32x3_split_a(A.data_ptr(), M, K, K, ap_.data_ptr(), st), "sa")
        _lib.check(lib.elv_tf32x3_split_b(B.data_ptr(), K, N, N, bp_.data_ptr(), st), "sb")
        _lib.check(lib.elv_tf32x3_gemm_planes(ap_.data_ptr(), bp_.data_ptr(), C.data_ptr(), M, N, K, N, st), "g")
torch.cuda.synchronize()
