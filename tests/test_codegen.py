"""CPU: the generic lowered-term -> CUDA compiler generates sources that NVRTC
compiles for sm_100a (no GPU needed), for every program in the corpus."""

import pytest

from paper_2002_02268_b200 import binomial, codegen, schedules
from paper_2002_02268_b200._ref import S

CHAIN = """
def chain = fun(x : 8.f32 => x |> map(fun(a => add(a)(a))) |> map(fun(b => mult(b)(b))) |> map(fun(c => add(c)(1.0))));
"""
MM_BT = """
def mmbt = fun(a : 6.5.f32 => fun(bt : 7.5.f32 =>
  a |> map(fun(r => bt |> map(fun(c => dot(r, c)))))));
"""


def corpus():
    s = S()
    out = {"mm_highlevel": schedules.mm(8, 12, 16), "chain": s.ir.parse(CHAIN),
           "mm_bt": s.ir.parse(MM_BT)}
    for n in schedules.SCHEDULE_NAMES:
        out[n] = schedules.apply(n, 64, 32, 16).term
    for n in binomial.SCHEDULE_NAMES:
        out["bf_" + n] = binomial.apply(n, 5, 9)
    # a user schedule the templates do not know: tile(16,16) without reorder
    st, nf, tv, rules = s.strategy, s.normal_forms, s.traversals, s.rules
    user = st.seq(nf.dfnf_seq(tv.top_down(schedules.tile(16, 16)),
                              tv.top_down(st.seq(tv.is_reduce, rules.make_split(2)))), nf.LOWER_TO_C)
    out["user_tile16"] = st.run_strategy(user, schedules.mm(32, 48, 8))[0].term
    return out


@pytest.mark.parametrize("name,term", list(corpus().items()))
def test_generated_source_compiles(name, term):
    pytest.importorskip("cuda.bindings.nvrtc")
    c = codegen.compile_term(term)
    assert "elv_generated" in c.source
    cubin = codegen.nvrtc_cubin(c)
    assert len(cubin) > 1000


def test_shapes_and_errors():
    s = S()
    c = codegen.compile_term(schedules.apply("blocking", 64, 32, 16).term)
    assert c.in_shapes == ((64, 16), (16, 32)) and c.out_shape == (64, 32)
    bad = s.ir.parse("def f = fun(a : 4.f32 => zip(a)(a));")          # result is pairs
    with pytest.raises(codegen.CodegenError):
        codegen.compile_term(bad)
    illtyped = schedules.apply("blocking", 64, 64, 1031).term
    with pytest.raises(codegen.CodegenError):
        codegen.compile_term(illtyped)
