"""One small launch of every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck --error-exitcode 1 python scripts/sanitize_run.py

Odd shapes exercise the predicated tails; the host pipeline runs with a
forced ragged tiling.  Results are also checked against the f64 oracle so a
sanitizer run doubles as a parity run."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import oracle  # noqa: E402
from paper_2002_02268_b200 import binomial, interp, schedules, synth  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    quick = "--quick" in sys.argv
    shapes = [(129, 257, 33), (129, 300, 520)] if quick else [(129, 257, 33), (257, 1031, 513)]
    names = list(schedules.SCHEDULE_NAMES) + ["parallel_tf32x3", "parallel_fp16x3"]
    for (M, N, K) in shapes:
        A = synth.matrix(M, K, 5, 0)
        B = synth.matrix(K, N, 5, 1)
        ref, ab = oracle.mm_f64(A, B), oracle.absprod_np(A, B)
        for v in names:
            sched, tf = ("parallel", True) if v.startswith("parallel_") else (v, False)
            term = schedules.apply_padded(sched, M, N, K).term
            C = interp.run_tensor(term, torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), tf32x3=tf,
                                  tc_encoding="fp16" if v == "parallel_fp16x3" else "tf32")
            torch.cuda.synchronize()
            ok, worst = oracle.check(C.cpu().numpy(), ref, ab, K)
            print(f"{v:16s} {M}x{N}x{K} ok={ok} worst={worst:.3f}", flush=True)
            assert ok
    # mid-size, ragged: the cta_group::2 kernel by the pair / 1-CTA model (no env), guard rows included
    M, N, K = 1100, 2100, 600
    assert interp.pair_kernel(M, N)
    A = synth.matrix(M, K, 6, 0)
    B = synth.matrix(K, N, 6, 1)
    A[1099, 5] = 2.0 ** -110
    ref, ab = oracle.mm_f64(A, B), oracle.absprod_np(A, B)
    for enc in ("tf32", "fp16"):
        term = schedules.apply_padded("parallel", M, N, K).term
        C = interp.run_tensor(term, torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), tf32x3=True,
                              tc_encoding=enc)
        torch.cuda.synchronize()
        ok, worst = oracle.check(C.cpu().numpy(), ref, ab, K)
        print(f"mid-size pair {enc} {M}x{N}x{K} ok={ok} worst={worst:.3f}", flush=True)
        assert ok
    if os.environ.get("ELV_SERPENTINE") == "1":
        # more pair tiles than clusters (80 > 74): an odd wave walks its k-blocks backwards
        M, N, K = 2560, 2048, 512
        A = synth.matrix(M, K, 9, 0)
        B = synth.matrix(K, N, 9, 1)
        ref, ab = oracle.mm_f64(A, B), oracle.absprod_np(A, B)
        for enc in ("tf32", "fp16"):
            term = schedules.apply_padded("parallel", M, N, K).term
            C = interp.run_tensor(term, torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), tf32x3=True,
                                  tc_encoding=enc)
            torch.cuda.synchronize()
            ok, worst = oracle.check(C.cpu().numpy(), ref, ab, K)
            print(f"serpentine pair {enc} {M}x{N}x{K} ok={ok} worst={worst:.3f}", flush=True)
            assert ok
    # range guard: marked rows / columns recomputed by the fix-up (both encodings)
    M, N, K = 160, 200, 576
    A = synth.matrix(M, K, 8, 0)
    B = synth.matrix(K, N, 8, 1)
    A[7, 3] = 2.0 ** -110
    B[9, 11] = 2.0 ** -110
    ref, ab = oracle.mm_f64(A, B), oracle.absprod_np(A, B)
    for enc in ("tf32", "fp16"):
        term = schedules.apply_padded("parallel", M, N, K).term
        C = interp.run_tensor(term, torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), tf32x3=True,
                              tc_encoding=enc)
        torch.cuda.synchronize()
        ok, worst = oracle.check(C.cpu().numpy(), ref, ab, K)
        print(f"guarded {enc} ok={ok} worst={worst:.3f}", flush=True)
        assert ok
    # the C-ABI pipelined row shard at ndev = 1 (NCCL broadcast in chunks, split on arrival)
    import ctypes
    from paper_2002_02268_b200 import _lib
    lib = _lib.load()
    _lib.check(lib.elv_nccl_init(1, (ctypes.c_int * 1)(0)), "nccl_init")
    try:
        Ad, Bd = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
        for v in (6, 7, 8):
            P = torch.empty(lib.elv_pack_b_bytes(K, N) // 4, device=dev)
            C = torch.empty((M, N), device=dev)
            wsb = lib.elv_gemm_rowshard_workspace_bytes(v, M, N, K, 2)
            W = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
            vp = ctypes.c_void_p
            rc = lib.elv_gemm_rowshard_pipelined(v, 1, (ctypes.c_int * 1)(0), (vp * 1)(Ad.data_ptr()), Bd.data_ptr(),
                                                 (vp * 1)(P.data_ptr()), (vp * 1)(C.data_ptr()),
                                                 (ctypes.c_int * 1)(M), N, K, 2, (vp * 1)(W.data_ptr()), wsb,
                                                 (vp * 1)(torch.cuda.current_stream().cuda_stream))
            _lib.check(rc, "rowshard_pipelined")
            torch.cuda.synchronize()
            ok, worst = oracle.check(C.cpu().numpy(), ref, ab, K)
            print(f"rowshard_pipelined v{v} ok={ok} worst={worst:.3f}", flush=True)
            assert ok
    finally:
        lib.elv_nccl_destroy()
    # host pipeline (elv_gemm_host) with ragged tiles
    os.environ["ELV_HOST_TILES"] = "96,160"
    M, N, K = 200, 300, 70
    A = torch.from_numpy(synth.matrix(M, K, 6, 0)).pin_memory()
    B = torch.from_numpy(synth.matrix(K, N, 6, 1)).pin_memory()
    for v in ("parallel", "parallel_tf32x3", "loopPerm"):
        sched, tf = ("parallel", True) if v == "parallel_tf32x3" else (v, False)
        p = interp.plan(schedules.apply_padded(sched, M, N, K).term, [(M, K), (K, N)], tf, "tf32")
        out = torch.empty((M, N), pin_memory=True)
        interp.HostPipeline(p, dev)(A, B, out)
        ok, worst = oracle.check(out.numpy(), oracle.mm_f64(A.numpy(), B.numpy()),
                                 oracle.absprod_np(A.numpy(), B.numpy()), K)
        print(f"host pipeline {v:16s} ok={ok} worst={worst:.3f}", flush=True)
        assert ok
    # binomial filter kernels
    img = synth.matrix(67, 45, 7, 2)
    for name in binomial.SCHEDULE_NAMES:
        term = binomial.apply(name, 67, 45)
        out = interp.run(term, [torch.from_numpy(img).to(dev)])
        torch.cuda.synchronize()
        refb = oracle.bf_interp_f64(img, name)
        assert np.all(np.abs(out.cpu().numpy() - refb) <= oracle.bf_bound(img)), name
        print(f"binomial {name} ok", flush=True)
    # K7F: the 3xTF32 split inside the pair kernel (applies at >= 148 pair tiles,
    # or at any shape under ELV_TF32X3_PAIR=32, which the pair sanitizer pass sets)
    M, N, K = 384, 520, 200
    A = synth.matrix(M, K, 9, 0)
    B = synth.matrix(K, N, 9, 1)
    A[5, 7] = 2.0 ** -110
    ref, ab = oracle.mm_f64(A, B), oracle.absprod_np(A, B)
    Ad, Bd = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    if lib.elv_tf32x3_fused_ok(Ad.data_ptr(), K, Bd.data_ptr(), N, M, N):
        flags = torch.empty(M + N, dtype=torch.int32, device=dev)
        C = torch.empty((M, N), device=dev)
        _lib.check(lib.elv_tf32x3_gemm_fused(Ad.data_ptr(), K, Bd.data_ptr(), N, C.data_ptr(), N, M, N, K,
                                             flags.data_ptr(), st), "gemm_fused")
        bp = torch.empty(lib.elv_tf32x3_b_planes_bytes(N, K), dtype=torch.uint8, device=dev)
        _lib.check(lib.elv_tf32x3_split_b(Bd.data_ptr(), K, N, N, bp.data_ptr(), st), "split_b")
        C2 = torch.empty((M, N), device=dev)
        _lib.check(lib.elv_tf32x3_gemm_fused_a(Ad.data_ptr(), K, bp.data_ptr(), Bd.data_ptr(), N, C2.data_ptr(), N,
                                               M, N, K, flags.data_ptr(), st), "gemm_fused_a")
        torch.cuda.synchronize()
        for name, X in (("fused", C), ("fused_a", C2)):
            ok, worst = oracle.check(X.cpu().numpy(), ref, ab, K)
            print(f"K7F {name} ok={ok} worst={worst:.3f}", flush=True)
            assert ok
    else:
        print("K7F: not applicable at this shape without ELV_TF32X3_PAIR=32 (skipped)", flush=True)
    # generated kernels: shared-memory tile mode (a user schedule outside the templates)
    from paper_2002_02268_b200 import codegen
    from paper_2002_02268_b200._ref import S
    st_, nf, tv, rules = S().strategy, S().normal_forms, S().traversals, S().rules
    n = 256
    user = st_.seq(nf.dfnf_seq(tv.top_down(schedules.tile(16, 16)),
                               tv.top_down(st_.seq(tv.is_reduce, rules.make_split(2)))), nf.LOWER_TO_C)
    term = st_.run_strategy(user, schedules.mm(n, n, n))[0].term
    A = synth.matrix(n, n, 3, 0)
    B = synth.matrix(n, n, 3, 1)
    C = codegen.run(term, [torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)])
    torch.cuda.synchronize()
    assert codegen.kernel_for(term).c.mode.startswith("smem-tile")
    ok, worst = oracle.check(C.cpu().numpy(), oracle.mm_f64(A, B), oracle.absprod_np(A, B), n)
    print(f"codegen smem-tile ok={ok} worst={worst:.3f}", flush=True)
    assert ok
    print("sanitize_run: all paths ran")


if __name__ == "__main__":
    main()
