"""CPU: the binomial-filter path -- schedules, dispatch, oracle pinned to the
reference interpreter's outputs (tests/golden/bf_*.npz)."""

import json
import os

import numpy as np
import pytest

import oracle
from paper_2002_02268_b200 import binomial, synth
from paper_2002_02268_b200._ref import S

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(GOLD, "golden.json")))["bf_cases"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_bf_oracle_bit_exact_vs_reference_interpreter(case):
    z = np.load(os.path.join(GOLD, case["name"] + ".npz"))
    img = z["img"]
    assert np.array_equal(synth.matrix(case["H"], case["W"], case["seed"], 2), img)
    for name in binomial.SCHEDULE_NAMES:
        assert np.array_equal(oracle.bf_interp_f64(img, name), z[name]), name


def test_separability_is_exact_in_f64_for_these_weights():
    """separateDot only reassociates: naive and separated agree to f64 rounding."""
    img = synth.matrix(32, 48, 1, 2)
    a, b = oracle.bf_interp_f64(img, "naive"), oracle.bf_interp_f64(img, "separated")
    assert np.allclose(a, b, rtol=0, atol=1e-15)


def test_schedules_decode_and_structure():
    s = S()
    for name in binomial.SCHEDULE_NAMES:
        t = binomial.apply(name, 12, 20)
        assert s.normal_forms.is_fully_lowered(t)
        assert s.ir.format_type(s.typecheck.typecheck(t)) == "(12.20.f32 -> 12.20.f32)"
        v, H, W = binomial.decode(t)
        assert binomial.SCHEDULE_NAMES[v] == name and (H, W) == (12, 20)
        txt = s.ir.pretty(t)
        assert ("mapPar" in txt) == name.endswith("Par")
        # separateDot turns the 9-tap dot into 3 row dots with wh then one with wv
        assert ("[1.0, 2.0, 1.0]" in txt) == name.startswith("separated")


def test_decode_rejects_other_one_argument_programs():
    s = S()
    other = s.ir.parse("def f = fun(img : 4.4.f32 => img |> mapSeq(mapSeq(fun(x => add(x)(x)))));")
    with pytest.raises(s.interp.EvalError):
        binomial.decode(other)
    with pytest.raises(s.interp.EvalError):
        binomial.decode(binomial.bf(4, 4))            # not lowered
