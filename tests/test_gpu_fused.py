"""K7F: 3xTF32 with the operand split fused into the tcgen05 pair kernel.

The fused kernel reads raw fp32 A / B by TMA and splits them in shared memory
(hi = the tf32 truncation the MMA itself reads, lo = rna_tf32(x - hi)), so it
must give the SAME BITS as the planes path (split prepass + pair kernel), and
through it the same parity with the oracle (reference interp.py:84-89,
145-148: the f64 fold, tau = 1 sqrt(K) bound).
"""

import numpy as np
import pytest
import torch

import oracle
from paper_2002_02268_b200 import _lib, interp, schedules, synth

pytestmark = pytest.mark.gpu


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _inputs(M, N, K, seed, dev, lda=None, ldb=None):
    lda, ldb = lda or K, ldb or N
    Ab = torch.empty((M, lda), device=dev)
    Bb = torch.empty((K, ldb), device=dev)
    synth.fill_device(Ab, seed, 0)
    synth.fill_device(Bb, seed, 1)
    return Ab, Bb


def _planes(A, B, M, N, K, lda, ldb):
    lib = _lib.load()
    st = _stream()
    ap = torch.empty(lib.elv_tf32x3_a_planes_bytes(M, K), dtype=torch.uint8, device=A.device)
    bp = torch.empty(lib.elv_tf32x3_b_planes_bytes(N, K), dtype=torch.uint8, device=A.device)
    C = torch.full((M, N), float("nan"), device=A.device)
    _lib.check(lib.elv_tf32x3_split_a(A.data_ptr(), M, K, lda, ap.data_ptr(), st), "split_a")
    _lib.check(lib.elv_tf32x3_split_b(B.data_ptr(), K, N, ldb, bp.data_ptr(), st), "split_b")
    _lib.check(lib.elv_tf32x3_gemm_planes(ap.data_ptr(), bp.data_ptr(), C.data_ptr(), M, N, K, N, st), "planes")
    _lib.check(lib.elv_tc_fixup(7, ap.data_ptr(), bp.data_ptr(), A.data_ptr(), lda, B.data_ptr(), ldb, 0,
                                C.data_ptr(), N, M, N, K, st), "fixup")
    return C


def _fused_a(A, B, M, N, K, lda, ldb):
    """B split once (planes), A split inside the GEMM."""
    lib = _lib.load()
    st = _stream()
    bp = torch.empty(lib.elv_tf32x3_b_planes_bytes(N, K), dtype=torch.uint8, device=A.device)
    _lib.check(lib.elv_tf32x3_split_b(B.data_ptr(), K, N, ldb, bp.data_ptr(), st), "split_b")
    flags = torch.empty(M, dtype=torch.int32, device=A.device)
    C = torch.full((M, N), float("nan"), device=A.device)
    _lib.check(lib.elv_tf32x3_gemm_fused_a(A.data_ptr(), lda, bp.data_ptr(), B.data_ptr(), ldb, C.data_ptr(), N,
                                           M, N, K, flags.data_ptr(), st), "gemm_fused_a")
    return C


def _fused(A, B, M, N, K, lda, ldb):
    lib = _lib.load()
    assert lib.elv_tf32x3_fused_ok(A.data_ptr(), lda, B.data_ptr(), ldb, M, N) == 1
    flags = torch.empty(M + N, dtype=torch.int32, device=A.device)
    C = torch.full((M, N), float("nan"), device=A.device)
    _lib.check(lib.elv_tf32x3_gemm_fused(A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), N, M, N, K,
                                         flags.data_ptr(), _stream()), "gemm_fused")
    return C, flags


SHAPES = [
    (4096, 4096, 1024),      # 256 pair tiles, one wave + a bit
    (4000, 3900, 1000),      # ragged M, N and K (K tail inside a 32-k block)
    (3584, 3072, 200),       # K < 512: the lo.lo correction is on
    (8192, 8192, 2048),      # 1024 pair tiles: multi-wave, wave-synchronised producers
    (2304, 4352, 8),         # K shorter than one k-block
    (2048, 2048, 1024),      # 64 pair tiles: mid-size, the pair kernel by the SMEM/MMA model
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_fused_bitwise_equals_planes(cuda, shape):
    M, N, K = shape
    A, B = _inputs(M, N, K, 21, cuda)
    Cp = _planes(A, B, M, N, K, K, N)
    Cf, flags = _fused(A, B, M, N, K, K, N)
    Ca = _fused_a(A, B, M, N, K, K, N)
    torch.cuda.synchronize()
    assert int(flags.sum()) == 0
    assert torch.equal(Cf.view(torch.int32), Cp.view(torch.int32))
    assert torch.equal(Ca.view(torch.int32), Cp.view(torch.int32))


def test_fused_padded_leading_dimensions(cuda):
    M, N, K = 2560, 4096, 700
    lda, ldb = K + 12, N + 36
    A, B = _inputs(M, N, K, 5, cuda, lda, ldb)
    Cp = _planes(A, B, M, N, K, lda, ldb)
    Cf, _ = _fused(A, B, M, N, K, lda, ldb)
    torch.cuda.synchronize()
    assert torch.equal(Cf.view(torch.int32), Cp.view(torch.int32))


@pytest.mark.parametrize("kind", ["uniform", "nonneg", "wide"])
def test_fused_vs_oracle(cuda, kind):
    M, N, K = 4096, 4096, 2048
    A, B = _inputs(M, N, K, 3, cuda)
    if kind == "nonneg":
        A.abs_(); B.abs_()
    elif kind == "wide":
        g = torch.Generator(device=cuda).manual_seed(7)
        A *= torch.exp2(torch.randint(-20, 21, A.shape, device=cuda, generator=g).float())
        B *= torch.exp2(torch.randint(-20, 21, B.shape, device=cuda, generator=g).float())
    Cf, _ = _fused(A, B, M, N, K, K, N)
    rows = np.random.default_rng(1).choice(M, 48, replace=False)
    Ah = A[rows].cpu().numpy()
    Bh = B.cpu().numpy()
    ok, worst = oracle.check(Cf[rows].cpu().numpy(), oracle.mm_f64(Ah, Bh), oracle.absprod(Ah, Bh), K)
    assert ok, f"{kind}: worst err/bound {worst:.3g}"


def test_fused_range_guard_rows_and_columns(cuda):
    """Out-of-window elements (inf, nan, 0 < |x| < 2^-100) mark their row of A /
    column of B inside the fused kernel; the fix-up recomputes them with the
    SIMT fold -- the same bits as the planes path."""
    M, N, K = 4096, 4096, 512
    A, B = _inputs(M, N, K, 9, cuda)
    A[17, 3] = float("inf")
    A[300, 511] = 1e-35
    A[4095, 100] = float("nan")
    B[5, 33] = 3e-38
    B[200, 4000] = float("-inf")
    Cp = _planes(A, B, M, N, K, K, N)
    Cf, flags = _fused(A, B, M, N, K, K, N)
    Ca = _fused_a(A, B, M, N, K, K, N)
    torch.cuda.synchronize()
    ca = Ca.cpu().numpy()
    assert np.array_equal(np.isnan(ca), np.isnan(Cp.cpu().numpy()))
    fl = flags.cpu().numpy()
    assert set(np.nonzero(fl[:M])[0]) == {17, 300, 4095}
    assert set(np.nonzero(fl[M:])[0]) == {33, 4000}
    a, b = Cf.cpu().numpy(), Cp.cpu().numpy()
    assert np.array_equal(np.isnan(a), np.isnan(b))
    m = ~np.isnan(a)
    assert np.array_equal(a[m].view(np.int32), b[m].view(np.int32))
    # a guarded finite row equals the SIMT fmaf chain of the parallel schedule
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    keep = np.ones(N, bool); keep[[33, 4000]] = False     # columns holding 3e-38 / -inf
    ref = oracle.mm_f64(Ah[300:301], Bh[:, keep])
    ok, worst = oracle.check(a[300:301, keep], ref, oracle.absprod(Ah[300:301], Bh[:, keep]), K)
    assert ok, worst


def test_elv_gemm_variant7_with_fused_path(cuda, monkeypatch):
    """elv_gemm(7) with ELV_TF32X3_FUSED=1 (read per call) runs K7F: same bits
    as the planes API (the default path)."""
    monkeypatch.setenv("ELV_TF32X3_FUSED", "1")
    M, N, K = 4096, 4096, 1024
    A, B = _inputs(M, N, K, 2, cuda)
    term = schedules.apply("parallel", M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=True, tc_encoding="tf32")
    Cp = _planes(A, B, M, N, K, K, N)
    torch.cuda.synchronize()
    assert torch.equal(C.view(torch.int32), Cp.view(torch.int32))


def test_fused_not_applicable_is_refused(cuda):
    lib = _lib.load()
    A, B = _inputs(512, 512, 64, 0, cuda)
    assert lib.elv_tf32x3_fused_ok(A.data_ptr(), 64, B.data_ptr(), 512, 512, 512) == 0   # 4 pair tiles
    assert lib.elv_tf32x3_fused_ok(A.data_ptr() + 4, 64, B.data_ptr(), 512, 4096, 4096) == 0   # misaligned A
    flags = torch.empty(1024, dtype=torch.int32, device=cuda)
    C = torch.empty((512, 512), device=cuda)
    rc = lib.elv_tf32x3_gemm_fused(A.data_ptr(), 64, B.data_ptr(), 512, C.data_ptr(), 512, 512, 512, 64,
                                   flags.data_ptr(), _stream())
    assert rc == _lib.ELV_EINVAL
