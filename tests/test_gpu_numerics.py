"""fp32 safety of the tensor-core encodings (K7 3xTF32, K8 3xFP16) on
adversarial inputs, against the f64 oracle at the stated tolerance.

The reference evaluates `add`/`mult` in f64 on any float (reference
pkg/src/stratir/interp.py:145-148).  Two mechanisms keep the tcgen05 paths
inside the fp32 bound for every input class, not only U(-1,1):
  * chunked accumulation: each k-block accumulates into a fresh TMEM buffer
    (corrections first, hi.hi last) and the epilogue adds the chunks with
    round-to-nearest in registers -- the tensor core's round-toward-zero
    accumulate otherwise biases long sums (positive inputs: 10.9x tau=1 at
    K=8192 before, profiles/r2/tc_numerics_before_chunked.jsonl);
  * the range guard: rows of A / columns of B with elements outside the
    encoding's exact window are recomputed by the SIMT fix-up (bitwise the
    parallel schedule's SIMT kernel, K6).
"""

import os

import numpy as np
import pytest
import torch

import oracle
from paper_2002_02268_b200 import interp, schedules, synth

pytestmark = pytest.mark.gpu

CLASSES = ("uniform", "positive", "dominant", "outlier_rows", "outlier_cols", "huge", "tiny", "dynamic")
ENCODINGS = ("tf32", "fp16")
SHAPES = [(512, 768, 1024), (300, 520, 640), (1024, 1024, 4096),
          (2048, 2304, 1024)]      # mid-size: the cta_group::2 kernel (interp.pair_kernel)


def make(M, N, K, kind, dev, seed=5):
    A = torch.empty((M, K), device=dev)
    B = torch.empty((K, N), device=dev)
    synth.fill_device(A, seed, 0)
    synth.fill_device(B, seed, 1)
    g = torch.Generator(device="cpu").manual_seed(seed)
    if kind == "positive":                       # no cancellation: |C| = (|A||B|)
        A.abs_()
        B.abs_()
    elif kind == "dominant":                     # one product dominates each sum
        idx = torch.randint(0, K, (M,), generator=g).to(dev)
        A[torch.arange(M, device=dev), idx] *= 4096.0
    elif kind == "outlier_rows":                 # 2^32 outlier meeting zeros in B
        A[:, 0] = 2.0 ** 32
        B[0, :] = 0.0
    elif kind == "outlier_cols":
        B[:, 1] = 2.0 ** 40
        B[:, 1][torch.arange(K, device=dev) % 7 != 0] *= 2.0 ** -80
    elif kind == "huge":                         # |x| >= 2^101 in every row of A
        A *= 2.0 ** 110
        B *= 2.0 ** -110
    elif kind == "tiny":                         # row maxima below 2^-101
        A *= 2.0 ** -110
        B *= 2.0 ** 110
    elif kind == "dynamic":                      # every element scaled by 2^u, u in [-20, 20]
        A *= torch.pow(2.0, torch.randint(-20, 21, (M, K), generator=g).float()).to(dev)
        B *= torch.pow(2.0, torch.randint(-20, 21, (K, N), generator=g).float()).to(dev)
    return A, B


def _tc(term, A, B, enc):
    return interp.run_tensor(term, A, B, tf32x3=True, tc_encoding=enc)


def _worst(C, A, B, K, rows=None):
    if rows is not None:
        A = A[rows]
        C = C[rows]
    Ah, Bh = A.double().cpu().numpy(), B.double().cpu().numpy()
    ref, ab = oracle.mm_f64(Ah, Bh), oracle.absprod_np(Ah, Bh)
    Cd = C.double().cpu().numpy()
    assert np.isfinite(Cd).all()
    return float((np.abs(Cd - ref) / oracle.bound(K, ab)).max())


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("kind", CLASSES)
@pytest.mark.parametrize("enc", ENCODINGS)
def test_tensor_core_classes_within_tau(cuda, enc, kind, shape):
    """Every class at tau = 1 (oracle.default_tau), except `dominant`, where
    the sqrt(K) law itself breaks down (one product sets the sum, its
    roundings do not average): there the tensor-core result must be no
    worse than the SIMT kernel's on the same inputs (1.2x + 0.1 slack),
    and the SIMT kernel's own ratio is recorded."""
    M, N, K = shape
    A, B = make(M, N, K, kind, cuda)
    term = schedules.apply_padded("parallel", M, N, K).term
    C = _tc(term, A, B, enc)
    torch.cuda.synchronize()
    worst = _worst(C, A, B, K)
    if kind == "dominant":
        simt = _worst(interp.run_tensor(term, A, B, tf32x3=False), A, B, K)
        print(f"{enc} {kind} {shape}: tc {worst:.3g} simt {simt:.3g}")
        assert worst <= max(1.0, 1.2 * simt + 0.1), f"tc {worst:.3g} vs simt {simt:.3g}"
    else:
        print(f"{enc} {kind} {shape}: worst err/bound {worst:.3g}")
        assert worst <= 1.0, f"{enc} {kind}: worst err/bound {worst:.3g}"


@pytest.mark.parametrize("enc", ENCODINGS)
def test_guarded_rows_and_columns_equal_the_simt_kernel(cuda, enc):
    """Rows of A / columns of B holding an element outside both encodings'
    windows (|x| = 2^-110: below tf32's 2^-100 guard and 2^-110 below its row
    maximum for fp16) are recomputed by the fix-up with the SIMT kernel's
    arithmetic: bitwise the parallel schedule's K6 output there; the rest of
    C stays on the tensor cores (within tau)."""
    M, N, K = 640, 768, 1024
    A, B = make(M, N, K, "uniform", cuda, seed=9)
    rows, cols = [5, 77, 300, 639], [9, 200, 767]
    for r in rows:
        A[r, 10] = 2.0 ** -110
    for c in cols:
        B[20, c] = -(2.0 ** -110)
    term = schedules.apply("parallel", M, N, K).term
    C = _tc(term, A, B, enc)
    C6 = interp.run_tensor(term, A, B, tf32x3=False)
    torch.cuda.synchronize()
    assert torch.equal(C[rows], C6[rows])
    assert torch.equal(C[:, cols], C6[:, cols])
    others = torch.ones(M, dtype=torch.bool)
    others[rows] = False
    assert not torch.equal(C[others], C6[others])      # the tensor-core path ran elsewhere
    assert _worst(C, A, B, K) <= 1.0


@pytest.mark.parametrize("enc", ENCODINGS)
def test_huge_rows_stay_finite(cuda, enc):
    """Rows of A with |x| up to 2^126 against columns of B scaled down so
    every product is finite: the fp16 encoding's power-of-two scales stay
    normal (the exponent is clamped on the low side only) and the epilogue
    unscales in two exact steps, so nothing overflows to Inf."""
    M, N, K = 512, 512, 1024
    A, B = make(M, N, K, "uniform", cuda, seed=3)
    A[::3] *= 2.0 ** 126
    A[1::3] *= 2.0 ** 101
    B *= 2.0 ** -100
    term = schedules.apply("parallel", M, N, K).term
    C = _tc(term, A, B, enc)
    torch.cuda.synchronize()
    assert torch.isfinite(C).all()
    assert _worst(C, A, B, K) <= 1.0


@pytest.mark.parametrize("kind", ["positive", "dynamic", "outlier_rows"])
@pytest.mark.parametrize("enc", ENCODINGS)
def test_bench_shape_checksums_adversarial(cuda, enc, kind):
    """configs[3] at full size (32768^2 x 8192) on adversarial classes, every
    element accounted for through column and row checksums against f64 (see
    test_gpu_parity.test_bench_shape_checksums_cover_every_element), plus
    sampled rows element-wise."""
    M, N, K = 32768, 32768, 8192
    A, B = make(M, N, K, kind, cuda, seed=1)
    C = _tc(schedules.apply("parallel", M, N, K).term, A, B, enc)
    torch.cuda.synchronize()
    rows = torch.tensor([0, 1, 4097, 16384, 32767], device=cuda)
    Cs = C[rows].clone()
    col = C.double().sum(0)
    row = C.double().sum(1)
    del C
    torch.cuda.empty_cache()
    assert _worst(Cs, A[rows], B, K) <= 1.0
    Ad = A.double()
    col_ref = Ad.sum(0) @ B.double()
    row_ref = Ad @ B.double().sum(1)
    b = Ad.abs() @ B.double().abs()
    del Ad
    b *= oracle.default_tau(K) * K ** 0.5 * 2.0 ** -24
    col_lin, row_lin = b.sum(0), b.sum(1)
    b.square_()
    col_rss, row_rss = b.sum(0).sqrt(), b.sum(1).sqrt()
    del b
    torch.cuda.empty_cache()
    ce, re = (col - col_ref).abs(), (row - row_ref).abs()
    lin = max((ce / col_lin).max().item(), (re / row_lin).max().item())
    cr, rr = (ce / col_rss).max().item(), (re / row_rss).max().item()
    print(f"{enc} {kind}: checksum err / rss-bound: columns {cr:.3g}, rows {rr:.3g}; / linear bound {lin:.3g}")
    # even fully correlated, the elements' errors stay under a tenth of their bounds on average
    assert lin <= 0.1
    if kind != "positive":
        assert cr <= 1.0 and rr <= 1.0
    # positive inputs (no cancellation): each chunk's hi.hi MMAs round toward
    # zero, leaving a same-signed residue of ~2^-22 |C_ij| per element (4/sqrt(K)
    # of its bound at most); it does not average out in a sum of 32768
    # elements: 4-6x the root-sum-square of the bounds, 0.02-0.04 of their
    # linear sum (profiles/r2/numerics_chunked.log)


@pytest.mark.parametrize("enc", ENCODINGS)
@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (1000, 1031, 777), (130, 70, 516), (640, 768, 1024)],
                         ids=lambda s: "x".join(map(str, s)))
def test_small_problem_paths_bitwise(cuda, enc, shape, monkeypatch):
    """Small problems (the 1-CTA kernel by the pair / 1-CTA model): the 1-CTA GEMM runs the
    range-guard fix-up itself and, for 3xFP16 with K <= 1024, the prepare is
    one launch (k16_prep_fused, B column slabs in shared memory).  Both give
    the bits of the separate launches (ELV_TC_FIXUP_INKERNEL=0,
    ELV_FP16X3_FUSED_PREP=0), with guarded rows and columns present."""
    M, N, K = shape
    A, B = make(M, N, K, "uniform", cuda, seed=4)
    A[3, 1] = 2.0 ** -110
    A[M - 1, K - 1] = float("inf")
    B[0, 2] = -(2.0 ** -110)
    B[K // 2, N - 1] = float("nan")
    term = schedules.apply_padded("parallel", M, N, K).term
    outs = []
    for inker, fprep in (("1", "1"), ("0", "1"), ("1", "0"), ("0", "0")):
        monkeypatch.setenv("ELV_TC_FIXUP_INKERNEL", inker)
        monkeypatch.setenv("ELV_FP16X3_FUSED_PREP", fprep)
        outs.append(_tc(term, A, B, enc).view(torch.int32).clone())
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    C6 = interp.run_tensor(term, A, B, tf32x3=False)
    C = outs[0].view(torch.float32)
    for r in (3, M - 1):
        assert torch.equal(torch.nan_to_num(C[r], nan=7.0), torch.nan_to_num(C6[r], nan=7.0))
    for c in (2, N - 1):
        assert torch.equal(torch.nan_to_num(C[:, c], nan=7.0), torch.nan_to_num(C6[:, c], nan=7.0))


@pytest.mark.parametrize("enc", ENCODINGS)
def test_small_problem_fixup_with_padded_operands(cuda, enc):
    """The in-kernel range-guard fix-up reads A and B through their leading
    dimensions: strided (padded) operands give the bits of contiguous ones."""
    M, N, K = 768, 640, 1024
    Ab = torch.empty((M, K + 20), device=cuda)
    Bb = torch.empty((K, N + 36), device=cuda)
    synth.fill_device(Ab, 6, 0)
    synth.fill_device(Bb, 6, 1)
    A, B = Ab[:, :K], Bb[:, :N]
    A[11, 5] = 2.0 ** -110
    B[7, 300] = float("inf")
    term = schedules.apply("parallel", M, N, K).term
    C = _tc(term, A, B, enc)
    Cc = _tc(term, A.contiguous(), B.contiguous(), enc)
    torch.cuda.synchronize()
    assert torch.equal(torch.nan_to_num(C, nan=7.0), torch.nan_to_num(Cc, nan=7.0))
    C6 = interp.run_tensor(term, A.contiguous(), B.contiguous(), tf32x3=False)
    assert torch.equal(torch.nan_to_num(C[11], nan=7.0), torch.nan_to_num(C6[11], nan=7.0))
    assert torch.equal(torch.nan_to_num(C[:, 300], nan=7.0), torch.nan_to_num(C6[:, 300], nan=7.0))


@pytest.mark.parametrize("enc", ENCODINGS)
@pytest.mark.parametrize("pbn", ["64", "128"])
def test_narrow_pair_kernel_bitwise(cuda, enc, pbn, monkeypatch):
    """The narrow CTA-pair kernel for small problems (ELV_SMALL_PAIR, read per
    call; measured slower, so opt-in) gives the bits of the 1-CTA kernel,
    guarded rows / columns included (its own in-kernel fix-up)."""
    M, N, K = 1000, 1031, 777
    A, B = make(M, N, K, "uniform", cuda, seed=13)
    A[2, 3] = 2.0 ** -110
    B[4, 1030] = -(2.0 ** -110)
    term = schedules.apply_padded("parallel", M, N, K).term
    ref = _tc(term, A, B, enc).clone()
    monkeypatch.setenv("ELV_SMALL_PAIR", pbn)
    C = _tc(term, A, B, enc)
    torch.cuda.synchronize()
    assert torch.equal(C.view(torch.int32), ref.view(torch.int32))


_PAIR_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {repo!r})
from paper_2002_02268_b200 import interp, schedules, synth
M, N, K = {M}, {N}, {K}
A = torch.empty((M, K), device="cuda"); B = torch.empty((K, N), device="cuda")
synth.fill_device(A, 17, 0); synth.fill_device(B, 17, 1)
A[5, 7] = 2.0 ** -110; B[9, N - 1] = -(2.0 ** -110)
t = schedules.apply_padded("parallel", M, N, K).term
for enc in ("tf32", "fp16"):
    np.save({out!r} + enc + ".npy", interp.run_tensor(t, A, B, tf32x3=True, tc_encoding=enc).cpu().numpy())
"""


@pytest.mark.parametrize("shape", [(2048, 2048, 2048), (2000, 1800, 777), (1100, 4100, 600), (2048, 2000, 300)],
                         ids=lambda s: "x".join(map(str, s)))
def test_mid_size_pair_choice_bitwise(cuda, tmp_path, shape):
    """Mid-size problems (fewer 256x256 pair tiles than SMs) run the
    cta_group::2 kernel when its modelled mainloop is shorter than the 1-CTA
    kernel's (interp.pair_kernel mirrors the library's choice): the bits are
    the 1-CTA kernel's (ELV_TF32X3_PAIR=0, read once per process, so a
    subprocess each), ragged tiles and range-guarded rows / columns
    included, and sampled rows are within the oracle bound."""
    import subprocess
    import sys
    M, N, K = shape
    assert interp.pair_kernel(M, N)
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("default", "0"):
        out = str(tmp_path / f"c_{mode}_")
        env = dict(os.environ)
        env.pop("ELV_TF32X3_PAIR", None)
        if mode == "0":
            env["ELV_TF32X3_PAIR"] = "0"
        subprocess.run([sys.executable, "-c", _PAIR_SCRIPT.format(repo=repo, M=M, N=N, K=K, out=out)],
                       env=env, check=True, timeout=300)
        outs[mode] = {enc: np.load(out + enc + ".npy") for enc in ENCODINGS}
    A = torch.empty((M, K), device=cuda); B = torch.empty((K, N), device=cuda)
    synth.fill_device(A, 17, 0); synth.fill_device(B, 17, 1)
    A[5, 7] = 2.0 ** -110
    B[9, N - 1] = -(2.0 ** -110)
    rows = [0, 5, 9, 255, 256, M // 2, M - 1]
    for enc in ENCODINGS:
        assert np.array_equal(outs["default"][enc].view(np.int32), outs["0"][enc].view(np.int32)), enc
        C = torch.from_numpy(outs["default"][enc]).to(cuda)
        assert _worst(C, A, B, K, rows=rows) <= 1.0, enc
