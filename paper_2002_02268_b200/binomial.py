"""Binomial filter: the paper's image-processing case study on the B200.

Program (the reference ships no .rise
file, pyproject.toml:19): a 3x3 binomial stencil with clamped borders,

    img |> pad2D(1) |> slide2D(3, 1) |> map2D(fun(nbh => dot(join(w2d), join(nbh))))

with w2d = [1 2 1; 2 4 2; 1 2 1] / 16 (the 1/16 folded into the weights).
pad2D/slide2D/map2D/dot are the reference parser's macros (ir.py:637-662).

Schedules, all built from reference
objects -- `separateDot` is the reference rule `make_separate_dot`
(rules.py:485-513) with wh = [1, 2, 1] and wv = [1, 2, 1] / 16:

    naive         lowerToC                                   K: k_bf_naive
    naivePar      topDown(parallel) ; lowerToC               K: k_bf_band<false>
    separated     topDown(separateDot) ; lowerToC            K: k_bf_separated
    separatedPar  topDown(separateDot) ; topDown(parallel) ; lowerToC
                                                             K: k_bf_band<true>

`run(term, [img])` (via `interp.run`) decodes the term by exact match of
`ir.pretty` against these schedules at the term's size and launches
`elv_binomial` (include/elevate_b200.h); anything else is EvalError.
"""

from __future__ import annotations

import functools

from . import _lib
from ._ref import S

BF_SOURCE = """
def bf = fun(img : H.W.f32 =>
  img |> pad2D(1) |> slide2D(3, 1) |> map2D(fun(nbh =>
    dot(join([[0.0625, 0.125, 0.0625], [0.125, 0.25, 0.125], [0.0625, 0.125, 0.0625]]), join(nbh)))));
"""
W2D = ((0.0625, 0.125, 0.0625), (0.125, 0.25, 0.125), (0.0625, 0.125, 0.0625))
WH = (1.0, 2.0, 1.0)
WV = (0.0625, 0.125, 0.0625)

SCHEDULE_NAMES = ("naive", "naivePar", "separated", "separatedPar")
VARIANTS = {n: i for i, n in enumerate(SCHEDULE_NAMES)}


def bf(H: int, W: int):
    return S().ir.parse(BF_SOURCE, {"H": H, "W": W})


def separate_dot():
    s = S()
    return s.rules.make_separate_dot(s.ir.Lit(W2D), s.ir.Lit(WH), s.ir.Lit(WV))


def strategy(name: str):
    s = S()
    st, tv, rules, nf = s.strategy, s.traversals, s.rules, s.normal_forms
    sep = tv.top_down(separate_dot())
    par = tv.top_down(rules.parallel)
    return {
        "naive": nf.LOWER_TO_C,
        "naivePar": st.seq(par, nf.LOWER_TO_C),
        "separated": st.seq(sep, nf.LOWER_TO_C),
        "separatedPar": st.seq(sep, st.seq(par, nf.LOWER_TO_C)),
    }[name]


def apply(name: str, H: int, W: int):
    s = S()
    res, ctx = s.strategy.run_strategy(strategy(name), bf(H, W))
    if not isinstance(res, s.strategy.Success):
        raise ValueError(f"binomial schedule {name} failed: {res.strategy}")
    return res.term


@functools.lru_cache(maxsize=128)
def template_key(name: str, H: int, W: int) -> str:
    return S().ir.pretty(apply(name, H, W))


def term_shape(term):
    ir = S().ir
    if not isinstance(term, ir.Lam) or isinstance(term.body, ir.Lam):
        return None
    t = term.param_type
    dims = []
    while isinstance(t, ir.ArrType):
        dims.append(t.size)
        t = t.elem
    if len(dims) != 2 or t != ir.F32 or not all(isinstance(d, int) for d in dims):
        return None
    return dims[0], dims[1]


def decode(term):
    """(variant, H, W) for one of the four binomial schedules, else EvalError."""
    s = S()
    shp = term_shape(term)
    if shp is None:
        raise s.interp.EvalError("no B200 kernel for term: not a binomial-filter schedule")
    if not s.normal_forms.is_fully_lowered(term):
        raise s.interp.EvalError("no B200 kernel for term: not fully lowered")
    key = s.ir.pretty(term)
    for name in SCHEDULE_NAMES:
        if template_key(name, *shp) == key:
            return VARIANTS[name], shp[0], shp[1]
    raise s.interp.EvalError("no B200 kernel for term: not one of the binomial schedules")


def launch(variant: int, img, out, stream=None):
    import torch
    lib = _lib.load()
    H, W = img.shape
    stream = stream or torch.cuda.current_stream(img.device)
    with torch.cuda.device(img.device):
        rc = lib.elv_binomial(variant, img.data_ptr(), out.data_ptr(), H, W, img.stride(0), out.stride(0),
                              stream.cuda_stream)
    _lib.check(rc, f"elv_binomial[{SCHEDULE_NAMES[variant]}]")
    return out
