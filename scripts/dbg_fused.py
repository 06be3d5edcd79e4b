import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2002_02268_b200 import _lib, synth
lib = _lib.load(); dev = torch.device("cuda", 0)
M, N, K = 4096, 4096, 1024
A = torch.empty((M, K), device=dev); synth.fill_device(A, 21, 0)
B = torch.empty((K, N), device=dev); synth.fill_device(B, 21, 1)
st = torch.cuda.current_stream().cuda_stream
ap = torch.empty(lib.elv_tf32x3_a_planes_bytes(M, K), dtype=torch.uint8, device=dev)
bp = torch.empty(lib.elv_tf32x3_b_planes_bytes(N, K), dtype=torch.uint8, device=dev)
Cp = torch.full((M, N), float("nan"), device=dev)
lib.elv_tf32x3_split_a(A.data_ptr(), M, K, K, ap.data_ptr(), st)
lib.elv_tf32x3_split_b(B.data_ptr(), K, N, N, bp.data_ptr(), st)
lib.elv_tf32x3_gemm_planes(ap.data_ptr(), bp.data_ptr(), Cp.data_ptr(), M, N, K, N, st)
for dbg in (0, 1, 2, 3):
    os.environ["ELV_K7F_DBG"] = str(dbg)
    flags = torch.empty(M + N, dtype=torch.int32, device=dev)
    C = torch.full((M, N), float("nan"), device=dev)
    rc = lib.elv_tf32x3_gemm_fused(A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, M, N, K, flags.data_ptr(), st)
    torch.cuda.synchronize()
    c, p = C.cpu().numpy(), Cp.cpu().numpy()
    nan = np.isnan(c).reshape(M // 128, 128, N // 128, 128).any(axis=(1, 3))
    diff = (c != p).reshape(M // 128, 128, N // 128, 128).mean(axis=(1, 3))
    print("dbg", dbg, "rc", rc, "nan blocks", int(nan.sum()), "of", nan.size, "flags", int(flags.sum()))
    print("nan map rows(128):", np.nonzero(nan.any(axis=1))[0].tolist()[:40])
    print("nan map cols(128):", np.nonzero(nan.any(axis=0))[0].tolist()[:40])
    print("diff fraction per block (first 4x8):\n", np.round(diff[:4, :8], 3))
    bad = (c != p) & ~np.isnan(c)
    if bad.any():
        r, q = np.nonzero(bad)
        print("first mismatches:", list(zip(r[:8].tolist(), q[:8].tolist())), c[r[0], q[0]], p[r[0], q[0]])
