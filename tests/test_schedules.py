"""CPU: the schedule catalog and the strategy-to-kernel dispatch."""

import pytest

from paper_2002_02268_b200 import dispatch, schedules
from paper_2002_02268_b200._ref import S

NAMES = schedules.SCHEDULE_NAMES


@pytest.fixture(scope="module")
def terms():
    return {n: schedules.apply(n, 64, 96, 64) for n in NAMES}


def test_every_schedule_is_fully_lowered_and_well_typed(terms):
    s = S()
    for n, sc in terms.items():
        assert s.normal_forms.is_fully_lowered(sc.term), n
        ty = s.typecheck.typecheck(sc.term)
        assert s.ir.format_type(ty) == "(64.64.f32 -> (64.96.f32 -> 64.96.f32))", n


def test_rule_success_counts_are_ordered(terms):
    """SPEC acceptance #6 (qualitative Fig. rewrite-steps):
    baseline < blocking <= max(vectorized..parallel); packing-based
    schedules cost the most."""
    c = {n: sc.rule_successes for n, sc in terms.items()}
    assert c["baseline"] == 9
    assert c["baseline"] < c["blocking"] <= max(c[n] for n in NAMES[2:])
    assert min(c["arrayPacking"], c["cacheBlocks"], c["parallel"]) > max(
        c["blocking"], c["vectorized"], c["loopPerm"])


def test_rule_counts_are_size_independent():
    a = schedules.apply("parallel", 32, 32, 32).rule_successes
    b = schedules.apply("parallel", 1024, 2048, 512).rule_successes
    assert a == b


@pytest.mark.parametrize("name", NAMES)
def test_dispatch_decodes_each_schedule(terms, name):
    p = dispatch.decode(terms[name].term, [(64, 64), (64, 96)])
    assert p.schedule == name
    assert p.variant == dispatch.VARIANTS[name]
    assert (p.M, p.N, p.K) == (64, 96, 64) and not p.tails


def test_structural_witnesses(terms):
    """Analogue of SPEC acceptance #5: the low-level vocabulary each kernel
    implements is present in the decoded term."""
    f = {n: dispatch.features(terms[n].term) for n in NAMES}
    assert f["baseline"]["splits"] == {} and f["baseline"]["mapSeq"] == 2
    for n in NAMES[1:]:
        assert f[n]["splits"].get(32, 0) >= 2 and f[n]["splits"].get(4) == 1, n
    for n in ("vectorized", "loopPerm", "arrayPacking", "cacheBlocks", "parallel"):
        assert f[n]["mapVec"] == 1, n
    for n in ("arrayPacking", "parallel"):
        assert f[n]["toMem"] == 1, n                      # packedB
    assert f["cacheBlocks"]["toMem"] == 2                 # + the block accumulator (cache_write)
    assert f["cacheBlocks"]["reduceSeqUnroll"] == 1       # unroll(ki)
    # parallelizeCopy: the packing copy's outer loop is mapPar (TVM
    # s[packedB].parallel(x)); parallel adds the row-block loop (parallel(xo))
    for n in ("arrayPacking", "cacheBlocks"):
        assert f[n]["mapPar"] == 1, n
    assert f["parallel"]["mapPar"] == 2 and f["parallel"]["reduceSeqUnroll"] == 1
    assert all(f[n]["mapPar"] == 0 for n in NAMES[:4])
    assert all(f[n]["high_level"] == 0 for n in NAMES)


def test_tvm_loop_orders(terms):
    """SPEC acceptance #5 analogue: the reorder puts the k-chunk reduce (ko)
    above both in-tile maps, and the in-chunk reduce (ki) above xi for
    blocking (xo,yo,ko,ki,xi,yi) but below it for loopPerm (xo,yo,ko,xi,ki,yi)."""
    ir = S().ir

    def ki_outside_xi(name):
        # in blocking the ki reduce's operator maps over whole (xi, yi) slices;
        # in loopPerm it sits inside the xi map and maps over yi only.
        txt = ir.pretty(terms[name].term)
        i = txt.index("reduceSeq", txt.index("reduceSeq") + 1)   # the ki reduce
        return "mapSeq(fun(" in txt[i:i + 60]
    assert ki_outside_xi("blocking") and ki_outside_xi("vectorized")
    assert not ki_outside_xi("loopPerm")
    for n in NAMES[1:]:
        f = dispatch.features(terms[n].term)
        assert f["reduceSeq"] + f["reduceSeqUnroll"] == 2, n      # ko and ki


def test_tf32x3_is_attached_to_parallel(terms):
    p = dispatch.decode(terms["parallel"].term, [(64, 64), (64, 96)], tf32x3=True)
    assert p.variant == 7 and p.variant_name == "parallel_tf32x3"
    with pytest.raises(S().interp.EvalError):
        dispatch.decode(terms["blocking"].term, [(64, 64), (64, 96)], tf32x3=True)


def test_dispatch_rejects_unlowered_and_foreign_terms():
    s = S()
    EvalError = s.interp.EvalError
    with pytest.raises(EvalError, match="not fully lowered"):
        dispatch.decode(schedules.mm(32, 32, 32))
    # a lowered program that is not one of the seven schedules
    other = s.ir.parse("def f = fun(a : 4.4.f32 => fun(b : 4.4.f32 => "
                       "a |> mapSeq(fun(r => b |> mapSeq(fun(c => r)))))); ")
    with pytest.raises(EvalError):
        dispatch.decode(other)
    # a transposed-operand variant (mm of B^T) must not be mistaken for mm
    odd = s.ir.parse("def f = fun(a : 4.4.f32 => fun(b : 4.4.f32 => a |> mapSeq(fun(r => "
                     "b |> mapSeq(fun(c => reduceSeq(fun(x => fun(y => add(x)(mult(fst(y))(snd(y))))))"
                     "(0.0)(zip(r)(c))))))));")
    with pytest.raises(EvalError):
        dispatch.decode(odd)


def test_padded_route_and_shape_mismatch():
    EvalError = S().interp.EvalError
    sc = schedules.apply_padded("parallel", 1000, 1000, 1000)
    assert (sc.M, sc.N, sc.K) == (1024, 1024, 1000)     # tile 32 on M/N, split(4) on K
    p = dispatch.decode(sc.term, [(1000, 1000), (1000, 1000)])
    assert p.tails and (p.M, p.N, p.K) == (1000, 1000, 1000)
    with pytest.raises(EvalError):
        dispatch.decode(sc.term, [(1000, 900), (1000, 1000)])    # inner sizes differ
    with pytest.raises(EvalError):
        dispatch.decode(sc.term, [(900, 1000), (1000, 1000)])    # not this term's padding


def test_reference_rules_fail_or_mistype_odd_shapes():
    """why the padded route exists."""
    s = S()
    with pytest.raises(ValueError):
        schedules.apply("arrayPacking", 1000, 1000, 1000)    # packB / interchange fail cleanly
    with pytest.raises(ValueError):
        schedules.apply("blocking", 257, 513, 1031)
    sc = schedules.apply("blocking", 64, 64, 1031)            # split(4) of K=1031 succeeds ...
    with pytest.raises(s.typecheck.TypeError_):
        s.typecheck.typecheck(sc.term)                         # ... but ill-typed (rules.py:207-210)
    # the ill-typed term is still decoded at its own (true) sizes
    p = dispatch.decode(sc.term, [(64, 1031), (1031, 64)])
    assert p.schedule == "blocking" and not p.tails
