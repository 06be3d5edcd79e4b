"""The seven TVM-tutorial GEMM schedules as strategies over the reference API.

The reference ships the leaf rules but not the composite schedules
(SPEC.md:449-516 specifies them; PAPER.md:269-315 lists them).  Each schedule
below is built *only* from reference objects (rules.py, traversals.py,
normal_forms.py, strategy.py) -- no rule is modified -- and yields a fully
lowered, well-typed term whose loop nest is the TVM tutorial's.
The output terms are the inputs of the hot path:
`paper_2002_02268_b200.interp.run` decodes them into one sm_100a kernel each.

`;;` is `dfnf_seq` (normal_forms.py:39-42).  Loop orders are outer -> inner
(x = rows of C, y = columns, k = reduction; o/i = tile / in-tile):

  schedule      strategy                                          TVM order
  baseline      DFNF ; topDown(fuseReduceMap) ; lowerToC          x, y, k            (271)
  blocking      tile(32,32) ;; split(4) ;; reorder_blocking       xo,yo,ko,ki,xi,yi  (26-30, 280-283)
  vectorized    blocking ;; vectorize(32) [lands on yi]           + vectorize(yi)    (33)
  loopPerm      tile ;; split(4) ;; reorder_loopperm ;; vec(32)   xo,yo,ko,xi,ki,yi  (37-42, 293-297)
  arrayPacking  packB ;; loopPerm ;; parallelizeCopy              + packedB          (49-63, 303-306)
  cacheBlocks   arrayPacking ;; topDown(isReduce;toMemAfter)
                ;; bottomUp(isAppliedReduce;unroll)               + cache_write, unroll(ki) (65-79)
  parallel      arrayPacking ;; topDown(parallel)
                ;; bottomUp(isAppliedReduce;unroll)               + parallel(xo)     (80-83, 313-314)

tile(x, y) is the paper's tileND: DFNF, fmap-recursive
blocking, function(split(n)) and `interchange`, here built from the shipped
interchange building blocks: at the row-block level,
`map(fun r => join(map g cb))` --mapFission--> `map(join)(map(fun r => map g
cb))` --mapMapInterchange--> `map(join)(transpose(map(fun c => map(fun r => g)
rows) cb))`, which moves the column-tile loop outside the in-tile row loop.

reorder ("non-trivial ... not discussed") is realised for the
two GEMM nests with shipped rules only: liftReduce (rules.py:328-358) twice
lifts the k-chunk reduce (ko) above xi and yi; absorbReduceInit
(rules.py:361-385) folds the per-chunk `0 + ...` into the running
accumulator; then liftReduce applied bottom-up lifts the in-chunk reduce (ki)
above yi (loopPerm) or above yi and xi (blocking).  Every schedule's
evaluation is therefore a sequential left fold acc + a_k b_k in k order (the
C oracle checks this bit-exactly against the reference interpreter).

`isAppliedReduce` is the reference's `predicate` combinator over a fully
applied reduce: the shipped `isReduce` also matches the bare `reduce`
primitive in function position, so `bottomUp(isReduce;unroll)` would unroll
the outer ko reduce instead of TVM's `unroll(ki)`.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass

from ._ref import S

# the `mm` program; pyproject.toml:19 names programs/*.rise
# but the file is not shipped, so the backend carries the source text.
MM_SOURCE = """
def mm = fun(a : M.K.f32 => fun(b : K.N.f32 =>
  a |> map(fun(arow => transpose(b) |> map(fun(bcol => dot(arow, bcol)))))));
"""

SCHEDULE_NAMES = ("baseline", "blocking", "vectorized", "loopPerm",
                  "arrayPacking", "cacheBlocks", "parallel")
ALIASES = {"parallelFull": "parallel"}

# divisibility each schedule's rules require: split(32) on rows and columns
# (tile / packB / vectorize(32) of the yi loop), split(4) on K.
REQUIRED_MULTIPLE = {
    "baseline": (1, 1, 1),
    "blocking": (32, 32, 4),
    "vectorized": (32, 32, 4),
    "loopPerm": (32, 32, 4),
    "arrayPacking": (32, 32, 4),
    "cacheBlocks": (32, 32, 4),
    "parallel": (32, 32, 4),
}


def mm(M: int, N: int, K: int):
    """Parse the mm program at concrete sizes (ir.py:680-683)."""
    s = S()
    return s.ir.parse(MM_SOURCE, {"M": M, "N": N, "K": K})


def _interchange():
    """tileND's interchange for the 2-D case: mapFission then
    mapMapInterchange one map level below the row-block map."""
    s = S()
    tv, rules, st = s.traversals, s.rules, s.strategy
    return tv.fmap(st.seq(rules.map_fission, tv.argument(rules.map_map_interchange)))


def _tile_nd(sizes):
    """tileND: DFNF, recursive fmap blocking innermost
    first, function(split(n.head)), interchange."""
    s = S()
    nf, tv, rules, st = s.normal_forms, s.traversals, s.rules, s.strategy
    if len(sizes) == 1:
        return st.seq(nf.DFNF, tv.function(rules.make_split(sizes[0])))
    return st.seq(nf.DFNF, tv.fmap(_tile_nd(sizes[1:])),
                  tv.function(rules.make_split(sizes[0])), nf.DFNF,
                  tv.top_down(_interchange()), nf.DFNF)


def tile(x: int, y: int):
    return _tile_nd([x, y])


def is_applied_reduce():
    s = S()
    ir = s.ir

    def pred(t):
        h, args = ir.spine(t)
        return isinstance(h, ir.Prim) and h.kind in ir.REDUCE_KINDS and len(args) == 3

    return s.strategy.predicate("isAppliedReduce", pred)


@functools.lru_cache(maxsize=None)
def _prefixes():
    s = S()
    nf, tv, rules, st = s.normal_forms, s.traversals, s.rules, s.strategy
    dseq = nf.dfnf_seq
    split4 = tv.top_down(st.seq(tv.is_reduce, rules.make_split(4)))
    lift = tv.top_down(rules.lift_reduce)
    lift_inner = tv.bottom_up(rules.lift_reduce)
    absorb = tv.top_down(rules.absorb_reduce_init)
    vec32 = tv.top_down(rules.make_vectorize(32))
    # tile, split k by 4, lift ko above yi and xi, fold the chunk init into acc
    tiled = dseq(dseq(dseq(dseq(tv.top_down(tile(32, 32)), split4), lift), lift), absorb)
    blocking = dseq(dseq(tiled, lift_inner), lift_inner)     # ki above yi and xi
    vectorized = dseq(blocking, vec32)
    loop_perm = dseq(dseq(tiled, lift_inner), vec32)          # ki above yi only
    # parallelizeCopy (undefined in paper and reference; TVM
    # s[packedB].parallel(x)): the outermost loop of the
    # packing copy inside toMem becomes mapPar.  The paper's extra
    # topDown(vectorize(32)) is meant for the copy's inner loop (TVM
    # s[packedB].vectorize(z)), but the shipped vectorize rule cannot type the
    # copy's identity function (rules.py:408-431 needs f : f32 -> f32 and the
    # identity is polymorphic), and a plain topDown lands on the k-products
    # map instead; the copy kernel (k_pack_b) moves 128-bit vectors anyway.
    parallelize_copy = tv.top_down(tv.argument_of("toMem", tv.top_down(rules.parallel)))
    array_packing = dseq(dseq(tv.top_down(rules.make_pack_b(32)), loop_perm), parallelize_copy)
    unroll_ki = tv.bottom_up(st.seq(is_applied_reduce(), rules.unroll))
    cache_blocks = dseq(dseq(array_packing,
                             tv.top_down(st.seq(tv.is_reduce, rules.to_mem_after))),
                        unroll_ki)
    parallel = dseq(dseq(array_packing, tv.top_down(rules.parallel)), unroll_ki)
    return {
        "baseline": st.seq(nf.DFNF, tv.top_down(rules.fuse_reduce_map)),
        "blocking": blocking,
        "vectorized": vectorized,
        "loopPerm": loop_perm,
        "arrayPacking": array_packing,
        "cacheBlocks": cache_blocks,
        "parallel": parallel,
    }


def canonical(name: str) -> str:
    name = ALIASES.get(name, name)
    if name not in SCHEDULE_NAMES:
        raise KeyError(f"unknown schedule {name!r}; known: {', '.join(SCHEDULE_NAMES)}")
    return name


def strategy(name: str):
    """The full schedule strategy `prefix ; lowerToC` (a reference Strategy)."""
    s = S()
    return s.strategy.seq(_prefixes()[canonical(name)], s.normal_forms.LOWER_TO_C)


@dataclass(frozen=True)
class Scheduled:
    name: str
    term: object          # the fully lowered stratir Expr
    M: int                # sizes the term was built at
    N: int
    K: int
    rule_successes: int   # ExecContext.total (strategy.py:62-67)


def apply(name: str, M: int, N: int, K: int) -> Scheduled:
    """Apply a named schedule to mm(M,N,K); raises on strategy Failure."""
    s = S()
    name = canonical(name)
    res, ctx = s.strategy.run_strategy(strategy(name), mm(M, N, K))
    if not isinstance(res, s.strategy.Success):
        raise ValueError(f"schedule {name} failed on mm({M},{N},{K}): {res.strategy}")
    return Scheduled(name, res.term, M, N, K, ctx.total)


def padded_shape(name: str, M: int, N: int, K: int):
    mM, mN, mK = REQUIRED_MULTIPLE[canonical(name)]
    up = lambda v, m: int(math.ceil(v / m) * m)
    return up(M, mM), up(N, mN), up(K, mK)


def apply_padded(name: str, M: int, N: int, K: int) -> Scheduled:
    """Apply the schedule at the smallest divisible shape >= (M,N,K).

    The reference rules reject (packB, rules.py:535-536) or mistype
    (splitJoin/splitReduce/vectorize, rules.py:176-183, 207-210, 439-440)
    non-divisible shapes, so odd shapes are scheduled at the padded shape and
    the backend runs the resulting term on the true-shape inputs with
    predicated tails.  Semantics: crop(eval(term, zero_pad(A), zero_pad(B))).
    """
    return apply(name, *padded_shape(name, M, N, K))


@functools.lru_cache(maxsize=256)
def template_key(name: str, M: int, N: int, K: int) -> str:
    """Canonical print (ir.py:332-360) of schedule(mm(M,N,K)); alpha-equal
    terms print identically, so this is the dispatch's match key."""
    s = S()
    res, _ = s.strategy.run_strategy(strategy(name), mm(M, N, K))
    if not isinstance(res, s.strategy.Success):
        return ""
    return s.ir.pretty(res.term)
