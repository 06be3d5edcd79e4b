"""GPU parity: every kernel variant against the oracle, through the C ABI.

Tolerance: |C - C_f64| <= sqrt(K) * 2^-24 * (|A||B|)_ij per
element, tau = 1 (oracle.check).  Golden cases compare against the reference
interpreter's own outputs; larger shapes against the f64 oracle.
"""

import json
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2002_02268_b200 import _lib, dispatch, interp, schedules, synth

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))
VARIANTS = list(schedules.SCHEDULE_NAMES) + ["parallel_tf32x3"]


def _sched(v):
    return ("parallel", True) if v.startswith("parallel_") else (v, False)


def _enc(v):
    """tc_encoding of a variant name (the library default is fp16)."""
    return "fp16" if v == "parallel_fp16x3" else "tf32"


def _device_inputs(M, N, K, seed, dev):
    A = torch.empty((M, K), device=dev, dtype=torch.float32)
    B = torch.empty((K, N), device=dev, dtype=torch.float32)
    synth.fill_device(A, seed, 0)
    synth.fill_device(B, seed, 1)
    return A, B


def test_native_library_is_what_runs(cuda):
    A, B = _device_inputs(64, 64, 64, 0, cuda)
    t = schedules.apply("parallel", 64, 64, 64).term
    interp.run_tensor(t, A, B)
    torch.cuda.synchronize()
    maps = open("/proc/self/maps").read()
    assert "libelevate_b200.so" in maps


def test_device_generator_matches_host(cuda):
    x = torch.empty(1 << 20, device=cuda)
    synth.fill_device(x, seed=3, tensor_id=1, offset=12345)
    assert np.array_equal(x.cpu().numpy(), synth.uniform(1 << 20, 3, 1, 12345))


@pytest.mark.parametrize("case", META["cases"], ids=[c["name"] for c in META["cases"]])
@pytest.mark.parametrize("tf32x3", [False, True], ids=["simt", "tf32x3"])
def test_golden_vs_reference_interpreter(cuda, case, tf32x3):
    if tf32x3 and case["schedule"] != "parallel":
        pytest.skip("3xTF32 is attached to the parallel schedule")
    z = np.load(os.path.join(GOLD, case["name"] + ".npz"))
    A, B, C_ref = z["A"], z["B"], z["C"]
    term = schedules.apply_padded(case["schedule"], case["M"], case["N"], case["K"]).term
    C = interp.run(term, [A, B], tf32x3=tf32x3)          # numpy in -> numpy out (host path)
    assert isinstance(C, np.ndarray) and C.shape == C_ref.shape
    ok, worst = oracle.check(C, C_ref, oracle.absprod(A, B), case["K"])
    assert ok, f"worst err/bound = {worst:.3g}"


def test_list_inputs_return_lists_like_the_reference(cuda):
    t = schedules.apply("baseline", 2, 3, 2).term
    B = [[1.5, -2.0, 0.25], [3.0, 0.5, -1.0]]
    C = interp.run(t, [[[1.0, 0.0], [0.0, 1.0]], B])     # mm(I, B) = B
    assert C == B
    t = schedules.apply("baseline", 1, 1, 3).term
    assert interp.run(t, [[[1.0, 2.0, 3.0]], [[4.0], [5.0], [6.0]]]) == [[32.0]]


@pytest.mark.parametrize("variant", VARIANTS)
def test_1024_cubed_vs_interpreter_arithmetic(cuda, variant):
    """configs[1]: every strategy at 1024^3 against the (bit-exact) C restatement
    of the interpreter's f64 arithmetic for that schedule."""
    name, tf = _sched(variant)
    M = N = K = 1024
    A, B = _device_inputs(M, N, K, 0, cuda)
    term = schedules.apply(name, M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=tf, tc_encoding=_enc(variant)).cpu().numpy()
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    ref = oracle.mm_interp_f64(Ah, Bh, name)
    ok, worst = oracle.check(C, ref, oracle.absprod_np(Ah, Bh), K)
    assert ok, f"{variant}: worst err/bound = {worst:.3g}"
    assert worst < 0.5


ODD = [(1000, 1000, 1000), (4096, 256, 4096), (257, 1031, 513), (1, 1, 1), (3, 5, 1),
       (129, 257, 17), (7, 300, 2048)]


@pytest.mark.parametrize("shape", ODD, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("variant", VARIANTS)
def test_odd_shapes_split_tails(cuda, shape, variant):
    """configs[4]: non-divisible shapes through the padded route (tails)."""
    name, tf = _sched(variant)
    M, N, K = shape
    A, B = _device_inputs(M, N, K, 11, cuda)
    term = schedules.apply_padded(name, M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=tf, tc_encoding=_enc(variant)).cpu().numpy()
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    ok, worst = oracle.check(C, oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh), K)
    assert ok, f"{variant} {shape}: worst err/bound = {worst:.3g}"


@pytest.mark.parametrize("variant", VARIANTS)
def test_strided_and_misaligned_operands(cuda, variant):
    """Leading dimensions larger than the row and 4-byte-misaligned bases
    force the scalar load paths of the same kernels."""
    name, tf = _sched(variant)
    M, N, K = 96, 160, 72
    big_a = torch.empty((M, K + 3), device=cuda); synth.fill_device(big_a, 5, 0)
    big_b = torch.empty((K, N + 5), device=cuda); synth.fill_device(big_b, 5, 1)
    A = big_a[:, 1:K + 1]          # base misaligned by 4 bytes, lda = K + 3
    B = big_b[:, 3:N + 3]
    p = dispatch.decode(schedules.apply(name, M, N, K).term, [(M, K), (K, N)], tf32x3=tf, tc_encoding=_enc(variant))
    out_big = torch.zeros((M, N + 1), device=cuda)
    C = interp.gemm(p, A, B, out=out_big[:, :N])
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    ok, worst = oracle.check(C.cpu().numpy(), oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh), K)
    assert ok, f"{variant}: worst err/bound = {worst:.3g}"
    assert torch.all(out_big[:, N] == 0)          # nothing written past the view


@pytest.mark.parametrize("variant", ["parallel", "parallel_tf32x3", "parallel_fp16x3", "cacheBlocks"])
def test_8192_cubed_row_sample(cuda, variant):
    """configs[2] roofline shape: sampled rows against the f64 oracle."""
    name, tf = _sched(variant)
    M = N = K = 8192
    A, B = _device_inputs(M, N, K, 2, cuda)
    term = schedules.apply(name, M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=tf, tc_encoding=_enc(variant))
    rows = torch.tensor([0, 1, 127, 128, 4095, 4096, 8190, 8191] + list(range(1000, 8000, 1111)),
                        device=cuda)
    Cs = C[rows].cpu().numpy()
    As = A[rows].cpu().numpy()
    Bh = B.cpu().numpy()
    ok, worst = oracle.check(Cs, oracle.mm_f64(As, Bh), oracle.absprod_np(As, Bh), K)
    assert ok, f"{variant}: worst err/bound = {worst:.3g}"


def test_pack_b_layout(cuda):
    K, N = 37, 100
    B = torch.empty((K, N), device=cuda); synth.fill_device(B, 1, 1)
    lib = _lib.load()
    P = torch.full((lib.elv_pack_b_bytes(K, N) // 4,), -7.0, device=cuda)
    _lib.check(lib.elv_pack_b(B.data_ptr(), P.data_ptr(), K, N, N, 32,
                              torch.cuda.current_stream().cuda_stream), "pack_b")
    Pn = P.cpu().numpy().reshape(-1, K, 32)           # [panel][k][c]
    Bp = np.zeros((K, Pn.shape[0] * 32), np.float32); Bp[:, :N] = B.cpu().numpy()
    expect = Bp.reshape(K, -1, 32).transpose(1, 0, 2)  # packedB[x][y][z] = B[y][32x+z]
    assert np.array_equal(Pn, expect)


def test_split_tf32(cuda):
    lib = _lib.load()
    x = torch.empty(1 << 16, device=cuda); synth.fill_device(x, 9, 0)
    x *= 1e3
    hi, lo = torch.empty_like(x), torch.empty_like(x)
    _lib.check(lib.elv_split_tf32(x.data_ptr(), hi.data_ptr(), lo.data_ptr(), x.numel(),
                                  torch.cuda.current_stream().cuda_stream), "split")
    h = hi.cpu().numpy().view(np.uint32)
    l = lo.cpu().numpy().view(np.uint32)
    assert np.all(h & 0x1FFF == 0) and np.all(l & 0x1FFF == 0)     # tf32-exact planes
    xs = x.cpu().numpy().astype(np.float64)
    err = np.abs(xs - (hi.cpu().numpy().astype(np.float64) + lo.cpu().numpy().astype(np.float64)))
    assert np.all(err <= np.abs(xs) * 2.0 ** -21)


def test_errors_raise_eval_error(cuda):
    from paper_2002_02268_b200._ref import S
    EvalError = S().interp.EvalError
    t = schedules.apply("parallel", 64, 64, 64).term
    A = torch.zeros((64, 32), device=cuda)
    B = torch.zeros((64, 64), device=cuda)
    with pytest.raises(EvalError):
        interp.run_tensor(t, A, B)
    with pytest.raises(EvalError):
        interp.run(t, [np.zeros((64, 64), np.float32)])


@pytest.mark.parametrize("variant", ["parallel", "parallel_tf32x3", "baseline", "blocking"])
def test_error_vs_k_sweep(cuda, variant):
    """The stated tolerance (oracle.bound: tau=1 for K>=32, 2 below) holds
    from K=1 to K=4096 on 128x128 outputs."""
    name, tf = _sched(variant)
    for K in (1, 2, 3, 4, 8, 16, 31, 32, 64, 1000, 4096):
        M = N = 128
        A, B = _device_inputs(M, N, K, 21, cuda)
        term = schedules.apply_padded(name, M, N, K).term
        C = interp.run_tensor(term, A, B, tf32x3=tf, tc_encoding=_enc(variant)).cpu().numpy()
        Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
        ok, worst = oracle.check(C, oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh), K)
        assert ok, f"{variant} K={K}: worst err/bound = {worst:.3g}"


@pytest.mark.parametrize("variant", ["parallel", "parallel_tf32x3", "parallel_fp16x3"])
def test_bench_shape_row_sample(cuda, variant):
    """configs[3] maximum size (32768 x 32768 x 8192, the bench workload):
    sampled rows and a column sample against the f64 oracle."""
    name, tf = _sched(variant)
    M, N, K = 32768, 32768, 8192
    A, B = _device_inputs(M, N, K, 0, cuda)
    term = schedules.apply(name, M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=tf, tc_encoding=_enc(variant))
    rows = torch.tensor([0, 255, 256, 16383, 16384, 32511, 32767], device=cuda)
    cols = torch.tensor([0, 1, 255, 256, 20000, 32767], device=cuda)
    Bh = B.cpu().numpy()
    As = A[rows].cpu().numpy()
    ok, worst = oracle.check(C[rows].cpu().numpy(), oracle.mm_f64(As, Bh), oracle.absprod_np(As, Bh), K)
    assert ok, f"{variant} rows: worst err/bound = {worst:.3g}"
    Ah = A.cpu().numpy()
    Bc = Bh[:, cols.cpu().numpy()]
    ok, worst = oracle.check(C[:, cols].cpu().numpy(), oracle.mm_f64(Ah, Bc), oracle.absprod_np(Ah, Bc), K)
    assert ok, f"{variant} cols: worst err/bound = {worst:.3g}"
    del C
    torch.cuda.empty_cache()


_TILE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {repo!r})
from paper_2002_02268_b200 import interp, schedules, synth
M, N, K = {M}, {N}, {K}
A = torch.empty((M, K), device="cuda"); B = torch.empty((K, N), device="cuda")
synth.fill_device(A, 11, 0); synth.fill_device(B, 11, 1)
t = schedules.apply_padded("parallel", M, N, K).term
np.save({out!r}, interp.run_tensor(t, A, B, tf32x3=True).cpu().numpy())
"""


@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (300, 1000, 200)], ids=lambda s: "x".join(map(str, s)))
def test_tf32x3_tile_widths_bitwise_identical(cuda, tmp_path, shape):
    """The 1-CTA tcgen05 kernel at N tiles 256 / 128 / 64 (ELV_TF32X3_BN,
    read once per process, so one subprocess each): per-element arithmetic
    does not depend on the tile width -- bitwise equal -- and within the
    oracle bound."""
    import subprocess
    import sys
    M, N, K = shape
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for bn in (256, 128, 64):
        out = str(tmp_path / f"c{bn}.npy")
        env = dict(os.environ, ELV_TF32X3_BN=str(bn), ELV_TF32X3_PAIR="0")
        subprocess.run([sys.executable, "-c", _TILE_SCRIPT.format(repo=repo, M=M, N=N, K=K, out=out)],
                       env=env, check=True, timeout=300)
        outs[bn] = np.load(out)
    assert np.array_equal(outs[256], outs[128]) and np.array_equal(outs[256], outs[64])
    A, B = synth.matrix(M, K, 11, 0), synth.matrix(K, N, 11, 1)
    ok, worst = oracle.check(outs[64], oracle.mm_f64(A, B), oracle.absprod_np(A, B), K)
    assert ok, worst


@pytest.mark.parametrize("variant", ["parallel", "parallel_tf32x3", "parallel_fp16x3"])
def test_output_beyond_2_pow_31_elements(cuda, variant):
    """Maximum-size edge: C with more than 2^31 elements (8.6 GB), so every
    row/column offset must be computed in 64 bits; rows at the far end
    checked against the f64 oracle."""
    M, N, K = 65536 + 128, 32768, 32
    assert M * N > 2 ** 31
    sched, tf = _sched(variant)
    A, B = _device_inputs(M, N, K, 12, cuda)
    term = schedules.apply_padded(sched, M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=tf, tc_encoding=_enc(variant))
    torch.cuda.synchronize()
    rows = [0, 65535, 65536, M - 1]
    Ah, Bh = A[rows].cpu().numpy(), B.cpu().numpy()
    ok, worst = oracle.check(C[rows].cpu().numpy(), oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh), K)
    assert ok, worst
    del C
    torch.cuda.empty_cache()


@pytest.mark.parametrize("variant", ["parallel", "parallel_tf32x3", "parallel_fp16x3"])
def test_bench_shape_checksums_cover_every_element(cuda, variant):
    """configs[3] at full size, every element accounted for: the column sums
    e^T C must match (e^T A) B and the row sums C e must match A (B e) in
    f64.  Per-element errors are independent and centred, so a column sum's
    error is compared with the root-sum-square of its elements' bounds
    b_ij = tau sqrt(K) 2^-24 (|A||B|)_ij (correct kernels sit at ~4 % of b,
    a dropped 3xTF32 correction at 7-29x b); the linear sum of the bounds is
    asserted too.  A checksum of checksums: size-independent, so it runs at
    32768^2 x 8192 where the element-wise oracle cannot (torch f64 on the
    GPU is the checker here)."""
    name, tf = _sched(variant)
    M, N, K = 32768, 32768, 8192
    A, B = _device_inputs(M, N, K, 1, cuda)
    C = interp.run_tensor(schedules.apply(name, M, N, K).term, A, B, tf32x3=tf,
                          tc_encoding="fp16" if variant == "parallel_fp16x3" else "tf32")
    torch.cuda.synchronize()
    col = C.double().sum(0)
    row = C.double().sum(1)
    del C
    torch.cuda.empty_cache()
    Ad, Bd = A.double(), B.double()
    del A, B
    col_ref, row_ref = Ad.sum(0) @ Bd, Ad @ Bd.sum(1)
    b = Ad.abs() @ Bd.abs()                              # (|A||B|), f64
    b *= oracle.default_tau(K) * K ** 0.5 * 2.0 ** -24
    col_lin, row_lin = b.sum(0), b.sum(1)
    b.square_()
    col_rss, row_rss = b.sum(0).sqrt(), b.sum(1).sqrt()
    del b
    torch.cuda.empty_cache()
    ce, re = (col - col_ref).abs(), (row - row_ref).abs()
    assert (ce / col_lin).max().item() <= 1.0 and (re / row_lin).max().item() <= 1.0
    col_ratio, row_ratio = (ce / col_rss).max().item(), (re / row_rss).max().item()
    print(f"{variant}: checksum err / rss-bound: columns {col_ratio:.3g}, rows {row_ratio:.3g}")
    assert col_ratio <= 1.0, f"{variant}: column checksum err/rss-bound {col_ratio:.3g}"
    assert row_ratio <= 1.0, f"{variant}: row checksum err/rss-bound {row_ratio:.3g}"


FP16X3_SHAPES = [(4096, 4096, 512), (3200, 5000, 1000), (4100, 4700, 2049), (8192, 8192, 8192),
                 (1024, 1024, 1024), (300, 1000, 600), (129, 257, 513), (2048, 2048, 2048)]


@pytest.mark.parametrize("shape", FP16X3_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_fp16x3_vs_oracle(cuda, shape):
    """The 3xFP16 encoding (variant 8) where it applies (K >= 512): the
    cta_group::2 kernel (>= one wave of pair tiles) and the 1-CTA kernel at
    N tiles 64 / 128 / 256, ragged M/N/K: sampled rows and columns against
    the f64 oracle, same tau as every other kernel."""
    M, N, K = shape
    A, B = _device_inputs(M, N, K, 13, cuda)
    term = schedules.apply_padded("parallel", M, N, K).term
    p = interp.plan(term, [(M, K), (K, N)], True, "fp16")
    assert p.variant == 8
    C = interp.run_tensor(term, A, B, tf32x3=True, tc_encoding="fp16")
    rows = torch.tensor(sorted({0, 1, min(255, M - 1), min(256, M - 1), M // 2, M - 1}), device=cuda)
    As, Bh = A[rows].cpu().numpy(), B.cpu().numpy()
    ok, worst = oracle.check(C[rows].cpu().numpy(), oracle.mm_f64(As, Bh), oracle.absprod_np(As, Bh), K)
    assert ok, f"rows: worst {worst:.3g}"
    cols = torch.tensor(sorted({0, min(255, N - 1), min(256, N - 1), N - 1}), device=cuda)
    Ah, Bc = A.cpu().numpy(), Bh[:, cols.cpu().numpy()]
    ok, worst = oracle.check(C[:, cols].cpu().numpy(), oracle.mm_f64(Ah, Bc), oracle.absprod_np(Ah, Bc), K)
    assert ok, f"cols: worst {worst:.3g}"


def test_fp16x3_scaled_and_special_rows(cuda):
    """Per-row / per-column power-of-two scaling: rows and columns scaled by
    2^-60 .. 2^60 stay within the bound, an all-zero row gives exact zeros,
    and shapes below the applicability threshold fall back to 3xTF32."""
    M, N, K = 4096, 4096, 1024
    A, B = _device_inputs(M, N, K, 14, cuda)
    g = torch.Generator().manual_seed(3)
    A *= torch.pow(2.0, torch.randint(-60, 61, (M, 1), generator=g).float()).to(cuda)
    B *= torch.pow(2.0, torch.randint(-60, 61, (1, N), generator=g).float()).to(cuda)
    A[7] = 0.0
    term = schedules.apply("parallel", M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=True, tc_encoding="fp16")
    assert torch.all(C[7] == 0)
    rows = torch.tensor([0, 5, 1000, M - 1], device=cuda)
    As, Bh = A[rows].double().cpu().numpy(), B.double().cpu().numpy()
    ok, worst = oracle.check(C[rows].cpu().numpy(), oracle.mm_f64(As, Bh), oracle.absprod_np(As, Bh), K)
    assert ok, worst
    small = schedules.apply("parallel", 256, 256, 256).term
    assert interp.plan(small, [(256, 256), (256, 256)], True, "fp16").variant == 8
    A2, B2 = _device_inputs(256, 256, 256, 15, cuda)
    ref = interp.run_tensor(small, A2, B2, tf32x3=True)                  # variant 7
    got = interp.run_tensor(small, A2, B2, tf32x3=True, tc_encoding="fp16")
    assert torch.equal(got, ref)                                        # same kernel below the threshold


@pytest.mark.parametrize("variant", ["parallel", "parallel_tf32x3", "parallel_fp16x3"])
def test_nan_and_inf_propagate_like_ieee(cuda, variant):
    """Special values follow the interpreter's IEEE arithmetic row/column-wise:
    a NaN in A row r makes all of C row r NaN; +inf in B column c (with a
    nonzero A row) makes that column non-finite; every other element is
    unaffected and within the bound."""
    name, tf = _sched(variant)
    M, N, K = 512, 512, 1024
    A, B = _device_inputs(M, N, K, 16, cuda)
    A[3, 100] = float("nan")
    B[200, 7] = float("inf")
    term = schedules.apply(name, M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=tf, tc_encoding=_enc(variant)).cpu().numpy()
    assert np.isnan(C[3]).all()
    assert not np.isfinite(C[:, 7]).any()
    mask_r = np.ones(M, bool); mask_r[3] = False
    mask_c = np.ones(N, bool); mask_c[7] = False
    Ah, Bh = A.cpu().numpy()[mask_r], B.cpu().numpy()[:, mask_c]
    ok, worst = oracle.check(C[mask_r][:, mask_c], oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh), K)
    assert ok, worst


@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (1000, 1031, 777), (333, 700, 2048), (260, 520, 2049),
                                   (130, 70, 516)],
                         ids=lambda s: "x".join(map(str, s)))
def test_fp16x3_warp_row_prepare_bitwise(cuda, shape, monkeypatch):
    """Short rows (K <= 2048) split one row per warp instead of one per block
    (mode 2: the row held in registers, float4 loads; mode 1: two scalar
    passes), and B's column maxima in slabs of 8..64 rows: bit-identical C
    in every mode, including a zero row, a scaled row, K not a multiple of 4
    (mode 2 falls back to 1) and K just past the threshold."""
    M, N, K = shape
    A, B = _device_inputs(M, N, K, 16, cuda)
    A[3] = 0.0
    A[5] *= 2.0 ** -50
    term = schedules.apply_padded("parallel", M, N, K).term
    outs = []
    for flag, slab in (("2", "0"), ("1", "0"), ("0", "64"), ("2", "8"), ("1", "16")):
        monkeypatch.setenv("ELV_FP16X3_WARP_ROWS", flag)
        monkeypatch.setenv("ELV_FP16X3_COLMAX_SLAB", slab)
        outs.append(interp.run_tensor(term, A, B, tf32x3=True, tc_encoding="fp16"))
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    assert torch.all(outs[0][3] == 0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", schedules.SCHEDULE_NAMES)
def test_ragged_b_and_shape_other_than_the_annotation(cuda, name):
    """Like the reference interpreter: a term scheduled at mm(64,64,64) runs
    on 32x96 . 96xN inputs (its split sizes divide them), and a ragged B is
    cut to its shortest row (transpose = zip(*m), interp.py:115-120)."""
    term = schedules.apply(name, 64, 64, 64).term
    A, B = synth.matrix(32, 96, 5, 0), synth.matrix(96, 160, 5, 1)
    Bl = B.tolist()
    Bl[7] = Bl[7][:128]
    C = np.array(interp.run(term, [A.tolist(), Bl]))
    assert C.shape == (32, 128)
    Bt = np.ascontiguousarray(B[:, :128])
    ok, worst = oracle.check(C, oracle.mm_f64(A, Bt), oracle.absprod_np(A, Bt), 96)
    assert ok, worst


@pytest.mark.gpu
@pytest.mark.parametrize("enc", ["tf32", "fp16"])
def test_tensor_core_variant_on_a_shape_other_than_the_annotation(cuda, enc):
    """The relaxed decode on the tcgen05 path: a parallel term scheduled at
    mm(128,128,512) evaluated on 64x512 . 512x96 device operands."""
    term = schedules.apply("parallel", 128, 128, 512).term
    A, B = _device_inputs(64, 96, 512, 31, cuda)
    C = interp.run_tensor(term, A, B, tf32x3=True, tc_encoding=enc).cpu().numpy()
    assert C.shape == (64, 96)
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    ok, worst = oracle.check(C, oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh), 512)
    assert ok, worst


def test_k6_bulk_copy_staging_is_bitwise(cuda, tmp_path):
    """k6_sgemm_bulk (ELV_K6_BULK=1, read once per process: TMA bulk copies of
    the packed panels + mbarriers instead of the cp.async ring) gives the
    bits of the default parallel-schedule SIMT kernel."""
    import subprocess
    import sys
    M, N, K = 4096, 2048, 256
    A, B = _device_inputs(M, N, K, 12, cuda)
    term = schedules.apply("parallel", M, N, K).term
    C = interp.run_tensor(term, A, B).cpu().numpy()
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (f"import sys; sys.path.insert(0, {repo!r})\n"
            "import numpy as np, torch\n"
            "from paper_2002_02268_b200 import interp, schedules, synth\n"
            f"M, N, K = {M}, {N}, {K}\n"
            "A = torch.empty((M, K), device='cuda'); synth.fill_device(A, 12, 0)\n"
            "B = torch.empty((K, N), device='cuda'); synth.fill_device(B, 12, 1)\n"
            "C = interp.run_tensor(schedules.apply('parallel', M, N, K).term, A, B)\n"
            f"np.save({str(tmp_path / 'c.npy')!r}, C.cpu().numpy())\n")
    env = dict(os.environ, ELV_K6_BULK="1")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
    Cb = np.load(tmp_path / "c.npy")
    assert np.array_equal(C.view(np.int32), Cb.view(np.int32))


@pytest.mark.parametrize("variant", ["parallel", "parallel_tf32x3", "parallel_fp16x3", "cacheBlocks"])
def test_gemmcall_graph_replay_bitwise(cuda, variant):
    """GemmCall.graph(): the call's launches (memsets, PDL-chained kernels)
    captured once and replayed give the bits of direct calls."""
    M, N, K = 1024, 768, 1024
    name, tf = _sched(variant)
    A, B = _device_inputs(M, N, K, 31, cuda)
    p = dispatch.decode(schedules.apply(name, M, N, K).term, [(M, K), (K, N)], tf32x3=tf, tc_encoding=_enc(variant))
    C = torch.empty((M, N), device=cuda)
    call = interp.GemmCall(p, A, B, C)
    ref = call().clone()
    g = call.graph()
    C.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(C, ref)


@pytest.mark.parametrize("variant,shape", [
    ("parallel", (1024, 1024, 1024)), ("cacheBlocks", (1024, 1024, 1024)), ("baseline", (512, 512, 512)),
    ("parallel_tf32x3", (1024, 1024, 1024)), ("parallel_fp16x3", (1024, 1024, 1024)),
    ("parallel_tf32x3", (2048, 2048, 1024)), ("parallel_fp16x3", (2048, 2048, 1024)),
    ("parallel_fp16x3", (1024, 1024, 256))], ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
def test_launch_count_claim_matches_the_profiler(cuda, variant, shape):
    """GemmCall.count_launches -- the per-call basis of the bench's
    `gpu_launches` -- equals the kernels the CUDA profiler (CUPTI, via
    torch.profiler) records for one call: 1-CTA vs pair kernel (in-kernel
    vs separate range-guard fix-up), the 3xFP16 two-kernel prepare, K < 512
    running the fp16 request as 3xTF32, the SIMT pack kernels."""
    M, N, K = shape
    name, tf = _sched(variant)
    A, B = _device_inputs(M, N, K, 41, cuda)
    p = dispatch.decode(schedules.apply(name, M, N, K).term, [(M, K), (K, N)], tf32x3=tf, tc_encoding=_enc(variant))
    C = torch.empty((M, N), device=cuda)
    call = interp.GemmCall(p, A, B, C)
    call()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        call()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
             and "elv" in e.name]
    assert len(names) == call.launches, (call.launches, names)


@pytest.mark.parametrize("variant", ["parallel_tf32x3", "parallel_fp16x3"])
def test_serpentine_k_order_opt_in(cuda, tmp_path, variant):
    """ELV_SERPENTINE=1 (an experiment, off by default): odd waves of the pair
    kernel walk the k-blocks backwards.  Results stay within the tau = 1
    bound of the f64 oracle; the first wave's tiles (even parity) keep the
    default bits, and later waves' bits differ (the knob is live)."""
    import subprocess
    import sys
    M, N, K = 8192, 8192, 1024                   # 1024 pair tiles: ~14 waves of 74
    name, tf = _sched(variant)
    enc = _enc(variant)
    A, B = _device_inputs(M, N, K, 23, cuda)
    term = schedules.apply(name, M, N, K).term
    C = interp.run_tensor(term, A, B, tf32x3=tf, tc_encoding=enc).cpu().numpy()
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (f"import sys; sys.path.insert(0, {repo!r})\n"
            "import numpy as np, torch\n"
            "from paper_2002_02268_b200 import interp, schedules, synth\n"
            f"M, N, K = {M}, {N}, {K}\n"
            "A = torch.empty((M, K), device='cuda'); synth.fill_device(A, 23, 0)\n"
            "B = torch.empty((K, N), device='cuda'); synth.fill_device(B, 23, 1)\n"
            f"C = interp.run_tensor(schedules.apply({name!r}, M, N, K).term, A, B, tf32x3={tf}, tc_encoding={enc!r})\n"
            f"np.save({str(tmp_path / 'c.npy')!r}, C.cpu().numpy())\n")
    env = dict(os.environ, ELV_SERPENTINE="1")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
    Cs = np.load(tmp_path / "c.npy")
    # wave 0 = tiles 0..73 of raster group 0 (8 m-tiles, n-major): rows < 2048, cols < 9 * 256
    assert np.array_equal(C[:2048, :2304].view(np.int32), Cs[:2048, :2304].view(np.int32))
    assert not np.array_equal(C.view(np.int32), Cs.view(np.int32))
    rows = slice(0, M, 61)
    Ah, Bh = A.cpu().numpy()[rows], B.cpu().numpy()
    ok, worst = oracle.check(Cs[rows], oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh), K)
    assert ok, f"serpentine {variant}: worst err/bound {worst:.3g}"
