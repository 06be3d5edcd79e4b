"""CPU: pin the oracle against the reference's own outputs (tests/golden/).

The golden fixtures were produced by the reference interpreter
(stratir.interp.run, reference interp.py:157-162) -- see make_golden.py.  The
C oracle must reproduce them BIT-EXACTLY (it restates the interpreter's f64
fold order per schedule), and the synthetic generator must reproduce the
stored inputs bit-exactly.
"""

import json
import os

import numpy as np
import pytest

import oracle
from paper_2002_02268_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))


@pytest.mark.parametrize("case", META["cases"], ids=[c["name"] for c in META["cases"]])
def test_oracle_bit_exact_vs_reference_interpreter(case):
    z = np.load(os.path.join(GOLD, case["name"] + ".npz"))
    A, B, C = z["A"], z["B"], z["C"]
    Mp, Np, Kp = case["term_shape"]
    # the padded route: zero-pad, evaluate, crop (schedules.apply_padded)
    Ap = np.zeros((Mp, Kp), np.float32); Ap[:A.shape[0], :A.shape[1]] = A
    Bp = np.zeros((Kp, Np), np.float32); Bp[:B.shape[0], :B.shape[1]] = B
    got = oracle.mm_interp_f64(Ap, Bp, case["schedule"])[:A.shape[0], :B.shape[1]]
    assert got.shape == C.shape
    assert np.array_equal(got, C), "oracle differs from the reference interpreter"


@pytest.mark.parametrize("case", META["cases"], ids=[c["name"] for c in META["cases"]])
def test_synth_reproduces_golden_inputs(case):
    z = np.load(os.path.join(GOLD, case["name"] + ".npz"))
    M, N, K, seed = case["M"], case["N"], case["K"], case["seed"]
    assert np.array_equal(synth.matrix(M, K, seed, 0), z["A"])
    assert np.array_equal(synth.matrix(K, N, seed, 1), z["B"])


def test_known_answers_from_spec():
    k = META["kats"]
    assert k["dot_1x3x1"] == [[32.0]]
    assert k["identity_2x3x2"]["C"] == k["identity_2x3x2"]["B"]
    A = np.array([[1, 2, 3]], np.float32)
    B = np.array([[4], [5], [6]], np.float32)
    assert oracle.mm_interp_f64(A, B)[0, 0] == 32.0


def test_sequential_fold_agrees_with_blas_within_f64():
    A = synth.matrix(16, 64, 3, 0)
    B = synth.matrix(64, 16, 3, 1)
    seq = oracle.mm_interp_f64(A, B, "parallel")
    assert np.allclose(seq, oracle.mm_f64(A, B), rtol=0, atol=1e-12)


def test_synth_is_exact_in_fp32_and_in_range():
    x = synth.uniform(100000, seed=0, tensor_id=0)
    assert x.dtype == np.float32
    assert x.min() >= -1.0 and x.max() < 1.0
    assert np.array_equal((x.astype(np.float64) * 2 ** 23).round(), x.astype(np.float64) * 2 ** 23)
    # offsets address the same stream
    assert np.array_equal(synth.uniform(10, 0, 0, 500), x[500:510])


def test_tolerance_catches_lost_lo_term():
    """A single-TF32 product (the lo term dropped) must violate the bound."""
    K = 1024
    A = synth.matrix(32, K, 1, 0)
    B = synth.matrix(K, 32, 1, 1)
    ref = oracle.mm_f64(A, B)
    ab = oracle.absprod_np(A, B)

    def tf32(x):
        u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
        u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)   # round-to-nearest(away), 10-bit mantissa
        return u.view(np.float32)

    one_tf32 = (tf32(A).astype(np.float64) @ tf32(B).astype(np.float64))
    ok, worst = oracle.check(one_tf32, ref, ab, K)
    assert not ok and worst > 5
    fp32 = (A @ B).astype(np.float32)
    ok, worst = oracle.check(fp32, ref, ab, K)
    assert ok and worst < 0.5
