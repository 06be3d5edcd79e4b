"""TEST INFRASTRUCTURE ONLY: the CPU oracle for the ELEVATE GEMM hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this package; the product (paper_2002_02268_b200/) never does, and
must fail loudly rather than fall back to it.

Contents
  * `mm_oracle.c` (-> liboracle_mm.so): bit-exact C restatement of the
    reference interpreter's f64 arithmetic for the seven scheduled mm terms
    (reference pkg/src/stratir/interp.py:84-89, 145-148); pinned against the
    reference interpreter's own outputs in tests/golden/ (made by
    tests/golden/make_golden.py, which imports the reference).
  * `mm_f64`: numpy f64 GEMM for shapes the C loop is too slow for.
  * `bound`/`check`: the parity tolerance of SURVEY.md §8(d).
  * `bf_interp_f64` / `bf_bound`: the same for the binomial-filter path.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle_mm.so")

# every schedule's evaluation is a sequential left fold over k (see mm_oracle.c)
SCHEDULES = ("baseline", "blocking", "vectorized", "loopPerm", "arrayPacking", "cacheBlocks",
             "parallel")

_lib = None


def build() -> str:
    src = os.path.join(HERE, "mm_oracle.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle_mm.so"], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        for fn in ("oracle_mm_seq_f64", "oracle_absprod_f64"):
            f = getattr(lib, fn)
            f.restype = None
            f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
        for fn in ("oracle_bf_naive_f64", "oracle_bf_separated_f64"):
            f = getattr(lib, fn)
            f.restype = None
            f.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int] * 2
        _lib = lib
    return _lib


def _call(name, A, B):
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    C = np.empty((M, N), np.float64)
    getattr(_load(), name)(A.ctypes.data, B.ctypes.data, C.ctypes.data, M, N, K)
    return C


def mm_interp_f64(A, B, schedule: str = "baseline") -> np.ndarray:
    """What interp.run(schedule(mm), [A, B]) returns, bit-exactly (f64)."""
    if schedule not in SCHEDULES:
        raise KeyError(schedule)
    return _call("oracle_mm_seq_f64", A, B)


def bf_interp_f64(img, schedule: str = "naive") -> np.ndarray:
    """What interp.run(binomial_schedule(bf), [img]) returns, bit-exactly."""
    img = np.ascontiguousarray(img, np.float32)
    H, W = img.shape
    out = np.empty((H, W), np.float64)
    fn = {"naive": "oracle_bf_naive_f64", "naivePar": "oracle_bf_naive_f64",
          "separated": "oracle_bf_separated_f64", "separatedPar": "oracle_bf_separated_f64"}[schedule]
    getattr(_load(), fn)(img.ctypes.data, out.ctypes.data, H, W)
    return out


def bf_bound(img, tau: float = 1.0) -> np.ndarray:
    """fp32 tolerance for the 9-tap stencil: tau * 9 * 2^-24 * (|w| * |img|)
    (the deterministic gamma_n bound for <= 12 roundings of non-negative
    weights; the weights sum to 1)."""
    a = np.abs(np.asarray(img, np.float64))
    p = np.pad(a, 1, mode="edge")
    H, W = a.shape
    w = np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]]) / 16.0
    mag = sum(w[i, j] * p[i:i + H, j:j + W] for i in range(3) for j in range(3))
    return tau * 9 * 2.0 ** -24 * mag


def absprod(A, B) -> np.ndarray:
    return _call("oracle_absprod_f64", A, B)


def mm_f64(A, B) -> np.ndarray:
    """Full-size f64 oracle (BLAS dgemm; f64 rounding << fp32 tolerance)."""
    return np.asarray(A, np.float64) @ np.asarray(B, np.float64)


def absprod_np(A, B) -> np.ndarray:
    return np.abs(np.asarray(A, np.float64)) @ np.abs(np.asarray(B, np.float64))


def default_tau(K: int) -> float:
    """tau = 1 for K >= 32; tau = 2 below.

    The sqrt(K) law is probabilistic: at K <= 8 even correctly rounded
    sequential fp32 FFMA reaches 1.23x the tau=1 bound on 65k outputs
    (measured on B200, scripts/tf32x3_numerics.py), because K-1 roundings of
    partial sums are not yet averaged.  From K = 32 on every kernel stays
    below 0.5 (SIMT) / 0.4 (3xTF32)."""
    return 1.0 if K >= 32 else 2.0


def bound(K: int, absAB: np.ndarray, tau: float | None = None) -> np.ndarray:
    """Per-element parity bound tau * sqrt(K) * 2^-24 * (|A||B|)_ij.

    Calibrated in SURVEY.md §8(d): sequential fp32 reaches ~0.1 of it at
    K=1024; a single TF32 product violates it by ~29x at K=1024 (measured)."""
    tau = default_tau(K) if tau is None else tau
    return tau * np.sqrt(K) * 2.0 ** -24 * absAB


def check(C, ref_f64, absAB, K: int, tau: float | None = None):
    """(ok, worst ratio err/bound) for a device result against the f64 oracle."""
    C = np.asarray(C, np.float64)
    err = np.abs(C - ref_f64)
    b = bound(K, absAB, tau)
    # exact-zero rows/cols of |A||B| (e.g. all-zero inputs) must match exactly
    ratio = np.where(b > 0, err / np.where(b > 0, b, 1.0), np.where(err > 0, np.inf, 0.0))
    worst = float(ratio.max()) if ratio.size else 0.0
    return worst <= 1.0, worst
