"""The seven TVM-tutorial GEMM schedules as strategies over the reference API.

The reference ships the leaf rules but not the composite schedules
(SPEC.md:449-516 specifies them; PAPER.md:269-315 lists them).  Each schedule
below is built *only* from reference objects (rules.py, traversals.py,
normal_forms.py, strategy.py) -- no rule is modified -- and yields a fully
lowered, well-typed term for divisible shapes.  The output terms are the
inputs of the hot path: `paper_2002_02268_b200.interp.run` decodes them into
one sm_100a kernel variant each.

Paper listing -> strategy here (`;;` = `dfnf_seq`, normal_forms.py:39-42):

  baseline     DFNF ; topDown(fuseReduceMap) ; lowerToC
  blocking     tile(32,32) ;; topDown(isReduce;split(4))
               ;; topDown(liftReduce) ; lowerToC
  vectorized   blocking-prefix ;; topDown(vectorize(32)) ; lowerToC PAPER.md:33,42
  loopPerm     tile ;; split(4) ;; liftReduce ;; liftReduce
               ;; topDown(vectorize(32)) ; lowerToC
  arrayPacking topDown(packB) ;; loopPerm-prefix ; lowerToC
  cacheBlocks  arrayPacking-prefix ;; topDown(isReduce;toMemAfter)
               ;; bottomUp(isReduce;unroll) ; lowerToC
  parallel     arrayPacking-prefix ;; topDown(parallel)
               ;; bottomUp(isReduce;unroll) ; lowerToC

`reorder(1,2,5,6,3,4)` / `reorder(1,2,5,3,6,4)` are not shipped by the
reference ("non-trivial ... not discussed").  The reduction
loops are moved outward over the spatial tile loops with the shipped
`liftReduce` (rules.py:328-358): once for blocking (k-chunks outside the
32-column tile loop), twice for loopPerm (outside both j loops), which is the
part of TVM's reorder that changes the arithmetic's data reuse.  A
TVM-faithful `reorder`/`interchange` is SURVEY.md §8(f) rank 1 ("next").

tileND follows the paper's listing: DFNF, recursive fmap
blocking innermost-first, then `function(split(n.head))`.  The trailing
`interchange(i)` is the same missing piece and is omitted, so tile(32,32)
strip-mines both output dimensions (loops io, ii, jo, ji).
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
# (tile / packB), split(4) on K (blocking), split(32) of the k-products
# (vectorize(32) lands on the zipped k pairs, rules.py:429-431).
REQUIRED_MULTIPLE = {
    "baseline": (1, 1, 1),
    "blocking": (32, 32, 4),
    "vectorized": (32, 32, 32),
    "loopPerm": (32, 32, 32),
    "arrayPacking": (32, 32, 32),
    "cacheBlocks": (32, 32, 32),
    "parallel": (32, 32, 32),
}


def mm(M: int, N: int, K: int):
    """Parse the mm program at concrete sizes (ir.py:680-683)."""
    s = S()
    return s.ir.parse(MM_SOURCE, {"M": M, "N": N, "K": K})


def _tile_nd(sizes):
    """tileND without the trailing interchange."""
    s = S()
    nf, tv, rules, st = s.normal_forms, s.traversals, s.rules, s.strategy
    if len(sizes) == 1:
        return st.seq(nf.DFNF, tv.function(rules.make_split(sizes[0])))
    return st.seq(nf.DFNF, tv.fmap(_tile_nd(sizes[1:])),
                  tv.function(rules.make_split(sizes[0])), nf.DFNF)


def tile(x: int, y: int):
    return _tile_nd([x, y])


@functools.lru_cache(maxsize=None)
def _prefixes():
    s = S()
    nf, tv, rules, st = s.normal_forms, s.traversals, s.rules, s.strategy
    dseq = nf.dfnf_seq
    split4 = tv.top_down(st.seq(tv.is_reduce, rules.make_split(4)))
    lift = tv.top_down(rules.lift_reduce)
    vec32 = tv.top_down(rules.make_vectorize(32))
    tiled = dseq(tv.top_down(tile(32, 32)), split4)
    blocking = dseq(tiled, lift)
    vectorized = dseq(blocking, vec32)
    loop_perm = dseq(dseq(dseq(tiled, lift), lift), vec32)
    array_packing = dseq(tv.top_down(rules.make_pack_b(32)), loop_perm)
    unroll = tv.bottom_up(st.seq(tv.is_reduce, rules.unroll))
    cache_blocks = dseq(dseq(array_packing,
                             tv.top_down(st.seq(tv.is_reduce, rules.to_mem_after))),
                        unroll)
    parallel = dseq(dseq(array_packing, tv.top_down(rules.parallel)), unroll)
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
