"""Strategy-to-kernel dispatch: recognise a rewritten `mm` term.

Input: a fully lowered stratir term (normal_forms.py:45-53) produced by one of
the seven schedules, plus the shapes of the arguments it is applied to.
Output: a `KernelPlan` naming the sm_100a kernel variant and the problem
sizes, or `EvalError` (interp.py:16) for anything else -- there is no CPU
fallback.

Recognition is two-step:
  1. a feature scan of the low-level vocabulary the lowering rules emit
     (mapPar, mapVec, toMem, reduceSeqUnroll, split(n); rules.py:391-456,
     516-549) proposes a schedule and records the structural witnesses the
     kernel implements (tile 32, k-chunk 4, vector width, packed B, unroll);
  2. the proposal is confirmed by exact match of the canonical print
     `ir.pretty(term)` (ir.py:332-360) against the schedule applied to
     mm(M,N,K) at the term's own sizes.  `pretty` renumbers binders, so
     alpha-equal terms match regardless of fresh-name counters.

Sizes come from the annotated outer binders `fun(a : M.K.f32 => fun(b :
K.N.f32 => ...))` (the parser keeps them, ir.py:585-597), so terms that the
reference rules leave ill-typed on non-divisible shapes are
still decoded.  A term built at the padded shape (schedules.apply_padded) is
accepted for true-shape arguments and runs with predicated tails.
"""

from __future__ import annotations

from collections import Counter
from dataclasses import dataclass, field

from . import schedules
from ._ref import S

VARIANTS = {
    "baseline": 0, "blocking": 1, "vectorized": 2, "loopPerm": 3,
    "arrayPacking": 4, "cacheBlocks": 5, "parallel": 6, "parallel_tf32x3": 7, "parallel_fp16x3": 8,
}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}


def EvalError(msg):
    return S().interp.EvalError(msg)


@dataclass(frozen=True)
class KernelPlan:
    schedule: str
    variant: int
    M: int
    N: int
    K: int
    term_shape: tuple           # (M, N, K) the term was scheduled at
    tails: bool                 # true shape smaller than term shape
    features: dict = field(default_factory=dict, compare=False)

    @property
    def variant_name(self) -> str:
        return VARIANT_NAMES[self.variant]


def features(term) -> dict:
    """Low-level vocabulary of a lowered term (the decode table input)."""
    ir = S().ir
    kinds = Counter()
    splits = Counter()
    for t in ir.subterms(term):
        if isinstance(t, ir.Prim):
            kinds[t.kind] += 1
            if t.kind == "split":
                splits[t.nats[0]] += 1
    return {
        "mapPar": kinds["mapPar"],
        "mapSeq": kinds["mapSeq"],
        "mapVec": kinds["mapVec"],
        "toMem": kinds["toMem"],
        "reduceSeq": kinds["reduceSeq"],
        "reduceSeqUnroll": kinds["reduceSeqUnroll"],
        "transpose": kinds["transpose"],
        "splits": dict(sorted(splits.items())),
        "high_level": kinds["map"] + kinds["reduce"],
    }


def _guess(f: dict) -> list:
    """Schedules consistent with the feature scan, most likely first."""
    if f["mapPar"] >= 2:                     # parallelizeCopy's + the row-block loop's
        return ["parallel"]
    if f["toMem"] >= 2:                      # packedB + the cache_write accumulator
        return ["cacheBlocks"]
    if f["toMem"]:
        return ["arrayPacking"]
    if f["mapVec"]:
        # blocking's reorder (ki above xi) leaves one more transpose than loopPerm's
        return ["vectorized", "loopPerm"] if f["transpose"] >= 6 else ["loopPerm", "vectorized"]
    if 4 in f["splits"]:
        return ["blocking"]
    return ["baseline"]


def term_shape(term):
    """(M, N, K) from the annotated outer binders of an mm-shaped term."""
    ir = S().ir
    if not (isinstance(term, ir.Lam) and isinstance(term.body, ir.Lam)):
        raise EvalError("no B200 kernel for term: expected fun(a => fun(b => ...))")
    ta, tb = term.param_type, term.body.param_type

    def dims(t):
        out = []
        while isinstance(t, ir.ArrType):
            out.append(t.size)
            t = t.elem
        return out, t

    (da, ea), (db, eb) = dims(ta), dims(tb)
    if (len(da) != 2 or len(db) != 2 or ea != ir.F32 or eb != ir.F32
            or not all(isinstance(x, int) for x in da + db)):
        # unannotated binders: fall back to whole-term inference
        try:
            ty = S().typecheck.typecheck(term)
        except S().typecheck.TypeError_ as e:
            raise EvalError(f"no B200 kernel for term: {e}") from None
        da, _ = dims(ty.arg) if hasattr(ty, "arg") else ([], None)
        db, _ = dims(ty.res.arg) if hasattr(ty, "res") and hasattr(ty.res, "arg") else ([], None)
        if len(da) != 2 or len(db) != 2:
            raise EvalError("no B200 kernel for term: not a matrix-matrix program")
    if da[1] != db[0]:
        raise EvalError(f"no B200 kernel for term: inner sizes {da[1]} != {db[0]}")
    return da[0], db[1], da[1]


def decode(term, arg_shapes=None, tf32x3: bool = False, tc_encoding: str = "tf32") -> KernelPlan:
    """Map a lowered term (and the argument shapes) to a kernel plan."""
    nf = S().normal_forms
    Mt, Nt, Kt = term_shape(term)
    if not nf.is_fully_lowered(term):
        raise EvalError("no B200 kernel for term: not fully lowered "
                        "(high-level map/reduce remains; apply lowerToC)")
    f = features(term)
    key = S().ir.pretty(term)
    name = None
    for cand in _guess(f) + [n for n in schedules.SCHEDULE_NAMES if n not in _guess(f)]:
        if schedules.template_key(cand, Mt, Nt, Kt) == key:
            name = cand
            break
    if name is None:
        raise EvalError("no B200 kernel for term: it is not one of the seven "
                        f"GEMM schedules at mm({Mt},{Nt},{Kt})")
    if arg_shapes is None:
        M, N, K = Mt, Nt, Kt
    else:
        (am, ak), (bk, bn) = arg_shapes
        if ak != bk:
            raise EvalError(f"zip of lengths {ak} and {bk}")
        M, N, K = am, bn, ak
        if (M, N, K) != (Mt, Nt, Kt):
            # the reference reads no sizes from the annotations at run time
            # (interp.py:50-149): a term evaluates at any shape its split
            # sizes divide -- the same fold, so the same kernel; a shape that
            # pads up to the term's is the odd-shape extension (apply_padded)
            pad = schedules.padded_shape(name, M, N, K)
            if pad != (M, N, K) and pad != (Mt, Nt, Kt):
                raise EvalError(
                    f"arguments {M}x{K} . {K}x{N} do not fit a term scheduled at "
                    f"mm({Mt},{Nt},{Kt})")
    variant = VARIANTS[name]
    if tf32x3:
        if name != "parallel":
            raise EvalError("the 3xTF32 tcgen05 variant is attached to the parallel schedule")
        if tc_encoding not in ("tf32", "fp16"):
            raise EvalError(f"unknown tensor-core encoding {tc_encoding!r} (tf32 | fp16)")
        variant = VARIANTS["parallel_tf32x3" if tc_encoding == "tf32" else "parallel_fp16x3"]
    return KernelPlan(name, variant, M, N, K, (Mt, Nt, Kt),
                      (M, N, K) != (Mt, Nt, Kt), f)
