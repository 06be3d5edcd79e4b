"""CPU: zero-extent GEMMs follow the reference interpreter's outcome.

`interp.run` answers these from the shapes alone (there is no arithmetic):
an A without rows gives [] (interp.py:80-83), a B without rows raises
`transpose of empty array` (interp.py:115-120), and a B without columns gives
M empty rows for the baseline schedule and the same EvalError for the tiled
ones.  The reference interpreter (baseline/_ref) is run beside it as the
checker on every (schedule, shape) whose term the reference rules can build.
No GPU is touched."""

import numpy as np
import pytest
import torch

from paper_2002_02268_b200 import interp, schedules
from paper_2002_02268_b200._ref import S

SHAPES = [(0, 32, 32), (32, 0, 32), (32, 32, 0), (0, 0, 0), (0, 0, 32), (0, 32, 0), (32, 0, 0),
          (3, 0, 5), (3, 5, 0), (0, 3, 5)]


def _outcome(fn):
    try:
        return ("ok", fn())
    except S().interp.EvalError as err:
        return ("EvalError", str(err))


@pytest.mark.parametrize("name", schedules.SCHEDULE_NAMES)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_zero_extent_matches_reference(name, shape):
    M, N, K = shape
    try:
        term = schedules.apply(name, M, N, K).term
    except ValueError:
        pytest.skip("the reference rules cannot schedule this shape")
    A = [[1.0] * K for _ in range(M)]
    B = [[2.0] * N for _ in range(K)]
    ref = _outcome(lambda: S().interp.run(term, [A, B]))
    got = _outcome(lambda: interp.run(term, [A, B]))
    assert got[0] == ref[0], (ref, got)
    if ref[0] == "ok":
        assert got[1] == ref[1]


@pytest.mark.parametrize("kind", ["numpy", "torch"])
def test_zero_rows_array_operands(kind):
    term = schedules.apply("parallel", 0, 32, 32).term
    A, B = np.zeros((0, 32), np.float32), np.ones((32, 32), np.float32)
    if kind == "torch":
        A, B = torch.from_numpy(A), torch.from_numpy(B)
    C = interp.run(term, [A, B])
    assert tuple(C.shape) == (0, 32)
    assert isinstance(C, np.ndarray if kind == "numpy" else torch.Tensor)


def test_zero_extent_rejects_foreign_terms():
    """Shape shortcuts apply only to the seven GEMM schedules."""
    ir = S().ir
    with pytest.raises(S().interp.EvalError):
        interp._empty_gemm(ir.Lam("a", None, ir.Lam("b", None, ir.Var("a"))), [[], []], None)


def test_ragged_b_is_cut_to_the_shortest_row():
    B = [[1.0, 2.0, 3.0], [4.0, 5.0], [6.0, 7.0, 8.0]]
    assert interp._truncate_ragged(B) == [[1.0, 2.0], [4.0, 5.0], [6.0, 7.0]]
    assert interp._truncate_ragged([[1.0], [2.0]]) == [[1.0], [2.0]]


def test_any_divisible_shape_decodes():
    """The reference evaluates a scheduled term at any shape its split sizes
    divide (sizes are not read from the annotations at run time)."""
    from paper_2002_02268_b200 import dispatch
    term = schedules.apply("parallel", 64, 64, 64).term
    p = dispatch.decode(term, [(32, 96), (96, 128)])
    assert (p.M, p.N, p.K) == (32, 128, 96)
    with pytest.raises(S().interp.EvalError):
        dispatch.decode(term, [(40, 96), (96, 128)])      # pads to (64, 128, 96), not the term's shape
