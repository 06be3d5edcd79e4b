"""General lowered-term -> CUDA compiler.

The template dispatch (`dispatch.py`, `binomial.py`) recognises the seven
GEMM schedules and the four binomial schedules and runs hand-written
kernels.  Every other well-typed program over the reference's primitive
vocabulary (ir.py:109-118) is compiled here into one CUDA kernel -- the GPU
analogue of the reference SPEC's codegen-c module (absent
from the reference):

  * views, not copies, for split / join / transpose / zip / fst / snd /
    slide / padClamp / asVector / asScalar (index arithmetic);
  * map, mapSeq, mapPar, mapSeqUnroll, mapVec: lazily indexed (the consumer's
    loop decides where the element is computed);
  * reduce / reduceSeq / reduceSeqUnroll: a sequential fold loop in the
    reference's order (interp.py:84-89).  An array-valued accumulator (the
    lifted reduces of the reordered GEMM schedules) whose operator is
    elementwise -- element e of op(acc)(x) reads acc only at e, checked on a
    symbolic element -- is folded per demanded element, so nested lifted
    reduces become one scalar fold per output in the schedule's own order;
    any other array accumulator is materialised (two per-thread buffers);
  * toMem / id: identity (values are views; materialisation is a
    performance choice, not semantics -- interp.py:143-144);
  * add / mult: fp32 (interp.py:145-148); an add of a product, the body of
    every reduce over zipped pairs (acc + a * b), is one explicit fmaf --
    the hand-written kernels' FFMA fold -- and nothing else is contracted
    (--fmad=false), so the host build (cpu_source) rounds identically.

Thread mapping: one thread per output scalar ("per-scalar") unless some
array accumulator had to be materialised -- then every scalar would rebuild
it, so the kernel is regenerated in destination-passing form: the result is
written following the term's own producer structure (maps are loops, the
outermost two of them the thread index; layout primitives transform the
destination; small computing maps are materialised per thread), and no value
is computed twice.  Kernels are built with NVRTC for sm_100a and cached per
canonical term print (ir.pretty); `cpu_source` wraps the same code for a
host compiler, which is how the CPU test suite checks it against the
reference interpreter.
"""

from __future__ import annotations

import functools
import itertools
import os
import random
import re
from dataclasses import dataclass
from typing import Callable

from ._ref import S

ARRAY_PRIMS_1 = {"split", "join", "transpose", "slide", "padClamp", "asVector", "asScalar"}


class CodegenError(Exception):
    pass


# ----------------------------------------------------------------------------
# values

@dataclass
class Scal:
    code: str


@dataclass
class Prod(Scal):
    """A product a * b not yet rounded: an `add` consuming it emits one
    fused multiply-add, like the hand-written kernels' FFMA k-loops."""
    a: str = ""
    b: str = ""


def _add(x, y):
    """add(x)(y): acc + a * b folds (the reduce bodies of every GEMM
    schedule) become fmaf(a, b, acc) -- one rounding per step, the same
    arithmetic as the template kernels (K0-K6 fold with FFMA) and closer to
    the interpreter's f64 than a separately rounded product."""
    if isinstance(y, Prod):
        return Scal(f"fmaf({y.a}, {y.b}, {x.code})")
    if isinstance(x, Prod):
        return Scal(f"fmaf({x.a}, {x.b}, {y.code})")
    return Scal(f"({x.code} + {y.code})")


class Pair:
    """A pair whose components are evaluated on first use (zip pairs an
    element of each array; fst/snd pick one -- the other is never indexed)."""

    def __init__(self, fa, fb):
        self._fa, self._fb = fa, fb

    @functools.cached_property
    def a(self):
        return self._fa()

    @functools.cached_property
    def b(self):
        return self._fb()


@dataclass
class Arr:
    size: int
    elem: Callable[[str], object]      # index code -> element value
    inner: tuple                        # sizes of the element's array levels (() for scalars)


@dataclass
class Fn:
    apply: Callable[[object], object]


def shape_of(v) -> tuple:
    if isinstance(v, Arr):
        return (v.size,) + v.inner
    if isinstance(v, Scal):
        return ()
    raise CodegenError("pairs have no array shape")


class Gen:
    def __init__(self):
        self.lines: list[str] = []
        self.indent = 1
        self.ids = itertools.count()
        self.dry = 0
        self.emitted = 0                 # statements emitted or (dry) that would be
        self.consts: list[str] = []
        self.decls: list[str] = []       # function-scope declarations (strict-map buffers)
        self.par_sizes: list[int] = []   # extents of the parallel (thread) index levels
        self.elementwise = True          # mode A: lifted array reduces fold per element
        self.strict_maps = False         # mode B: materialise small computing maps
        self.materialised = 0            # array reduces that had to be materialised
        self.grid: tuple = ()             # smem-tile mode: explicit 2-D grid of `block`-thread blocks
        self.block = 128
        self.probing = 0                 # >0 inside shape probes
        self.fold_depth = 0              # >0 inside a per-element fold

    def fresh(self, hint: str) -> str:
        return f"{hint}{next(self.ids)}"

    def emit(self, line: str) -> None:
        self.emitted += 1
        if not self.dry:
            self.lines.append("  " * self.indent + line)

    def open(self, line: str) -> None:
        self.emit(line)
        self.indent += 1

    def close(self) -> None:
        self.indent -= 1
        self.emit("}")

    def dry_run(self, thunk):
        """Evaluate for the shape only, emitting nothing."""
        self.dry += 1
        try:
            return thunk()
        finally:
            self.dry -= 1


def _fmt(x: float) -> str:
    r = repr(float(x))
    if "e" not in r and "." not in r and "inf" not in r and "nan" not in r:
        r += ".0"
    return r + "f"


# ----------------------------------------------------------------------------
# primitives

def _buffer_view(g: Gen, buf: str, shape: tuple, base: str = "0"):
    """A view over a flat row-major buffer."""
    if not shape:
        return Scal(f"{buf}[{base}]")
    stride = 1
    for d in shape[1:]:
        stride *= d
    return Arr(shape[0], lambda i: _buffer_view(g, buf, shape[1:], f"({base} + ({i}) * {stride})"),
               tuple(shape[1:]))


def _materialise(g: Gen, v, buf: str, shape: tuple) -> None:
    """Emit a loop nest writing every scalar of `v` into buf (row-major)."""
    idx = []

    def rec(val, dims, flat):
        if not dims:
            if not isinstance(val, Scal):
                raise CodegenError("only scalar arrays can be materialised")
            g.emit(f"{buf}[{flat}] = {val.code};")
            return
        i = g.fresh("m")
        g.open(f"for (int {i} = 0; {i} < {dims[0]}; ++{i}) {{")
        stride = 1
        for d in dims[1:]:
            stride *= d
        rec(val.elem(i), dims[1:], f"({flat} + {i} * {stride})")
        g.close()

    rec(v, shape, "0")


class NotElementwise(Exception):
    pass


_IDENT = re.compile(r"[A-Za-z_][A-Za-z_0-9]*")


@functools.lru_cache(maxsize=65536)
def _same_index(a: str, b: str) -> bool:
    """Do two generated index expressions (non-negative ints, + * / % min
    max) denote the same value?  Equal text, or equal under 16 random
    assignments of their variables (the layout algebra only produces
    affine / div / mod forms, e.g. ((q / 32) * 32 + q % 32) == q)."""
    if a == b:
        return True
    names = sorted((set(_IDENT.findall(a)) | set(_IDENT.findall(b))) - {"min", "max"})
    pa, pb = a.replace("/", "//"), b.replace("/", "//")
    rng = random.Random(hash((a, b)) & 0xFFFFFFFF)
    try:
        for _ in range(16):
            env = {n: rng.randrange(0, 4096) for n in names}
            env.update(min=min, max=max)
            if eval(pa, {"__builtins__": {}}, env) != eval(pb, {"__builtins__": {}}, env):
                return False
    except Exception:
        return False
    return True


def _sym_acc(g: Gen, shape: tuple, path: list, code: str, depth: int = 0):
    """The accumulator as seen by one output element's fold: only element
    `path` exists (as the scalar `code`); any other index raises (except in
    shape probes, which index with placeholders)."""
    if depth == len(shape):
        return Scal(code)

    def elem(i):
        if not g.probing and not _same_index(i, path[depth]):
            raise NotElementwise()
        return _sym_acc(g, shape, path, code, depth + 1)
    return Arr(shape[depth], elem, tuple(shape[depth + 1:]))


def _lazy_nd(shape: tuple, leaf, path=()):
    """An array value whose element at a full index path is leaf(path)."""
    if len(path) == len(shape):
        return leaf(list(path))
    return Arr(shape[len(path)], lambda i: _lazy_nd(shape, leaf, path + (i,)), tuple(shape[len(path) + 1:]))


def _fold_element(g: Gen, op: Fn, init, xs: Arr, shape: tuple, path: list):
    acc = g.fresh("acc")
    v0 = init
    for q in path:
        v0 = v0.elem(q)
    g.emit(f"float {acc} = {v0.code};")
    k = g.fresh("k")
    g.open(f"for (int {k} = 0; {k} < {xs.size}; ++{k}) {{")
    g.fold_depth += 1
    try:
        v = op.apply(_sym_acc(g, shape, path, acc)).apply(xs.elem(k))
        for q in path:
            v = v.elem(q)
    finally:
        g.fold_depth -= 1
    if not isinstance(v, Scal):
        raise CodegenError("reduce operator returned a non-scalar element")
    g.emit(f"{acc} = {v.code};")
    g.close()
    return Scal(acc)


def _is_elementwise(g: Gen, op: Fn, init, xs: Arr, shape: tuple) -> bool:
    """Does element e of op(acc)(x) read acc at e only?  Probed on symbolic
    indices in dry mode; then each demanded element of the reduce is its own
    scalar left fold -- the interpreter's order (interp.py:84-89) per element."""
    path = [f"__e{d}__" for d in range(len(shape))]
    try:
        g.dry_run(lambda: _fold_element(g, op, init, xs, shape, path))
    except NotElementwise:
        return False
    return True


def _lazy_reduce(g: Gen, op: Fn, init, xs: Arr, shape: tuple):
    return _lazy_nd(shape, lambda path: _fold_element(g, op, init, xs, shape, path))


def _reduce(g: Gen, op: Fn, init, xs: Arr):
    if isinstance(init, Scal):
        acc = g.fresh("acc")
        g.emit(f"float {acc} = {init.code};")
        k = g.fresh("k")
        g.open(f"for (int {k} = 0; {k} < {xs.size}; ++{k}) {{")
        v = op.apply(Scal(acc)).apply(xs.elem(k))
        if not isinstance(v, Scal):
            raise CodegenError("scalar reduce operator returned a non-scalar")
        g.emit(f"{acc} = {v.code};")
        g.close()
        return Scal(acc)
    if isinstance(init, Arr):
        shape = shape_of(init)
        # inside an element fold the enclosing check covers this reduce too
        # (it evaluates the whole nest at a symbolic element)
        if g.elementwise and (g.fold_depth > 0 or _is_elementwise(g, op, init, xs, shape)):
            return _lazy_reduce(g, op, init, xs, shape)
        g.materialised += 1
        n = 1
        for d in shape:
            n *= d
        # two buffers, swapped by pointer after every step
        ba, bb = g.fresh("accbuf"), g.fresh("accbuf")
        cur, nxt = g.fresh("cur"), g.fresh("nxt")
        g.emit(f"float {ba}[{n}], {bb}[{n}];")
        g.emit(f"float* {cur} = {ba}; float* {nxt} = {bb};")
        _materialise(g, init, cur, shape)
        k = g.fresh("k")
        g.open(f"for (int {k} = 0; {k} < {xs.size}; ++{k}) {{")
        v = op.apply(_buffer_view(g, cur, shape)).apply(xs.elem(k))
        _materialise(g, v, nxt, shape)
        g.emit(f"{{ float* sw = {cur}; {cur} = {nxt}; {nxt} = sw; }}")
        g.close()
        return _buffer_view(g, cur, shape)
    raise CodegenError("pair-valued reduce accumulators are not supported")


def _prim(g: Gen, p) -> object:
    k = p.kind
    if k in ("map", "mapSeq", "mapPar", "mapSeqUnroll", "mapVec"):
        def map_f(f):
            def map_xs(xs):
                if not isinstance(xs, Arr):
                    raise CodegenError(f"{k} expects an array")
                before = g.emitted
                g.probing += 1
                try:
                    probe = g.dry_run(lambda: f.apply(xs.elem("0")))
                finally:
                    g.probing -= 1
                emits = g.emitted > before
                elem_shape = _shape_or_scalar(probe)
                lazy = Arr(xs.size, lambda i: f.apply(xs.elem(i)), elem_shape)
                n = xs.size
                for d in elem_shape:
                    n *= d
                if g.strict_maps and emits and not isinstance(probe, Pair) and n <= STRICT_MAP_MAX:
                    # the body computes (a reduce): evaluate each element once into
                    # a per-thread buffer instead of once per consumer read
                    buf = g.fresh("mbuf")
                    g.emit(f"float {buf}[{n}];")
                    _write(g, lazy, _out_buffer(buf, (xs.size,) + elem_shape))
                    return _buffer_view(g, buf, (xs.size,) + elem_shape)
                return lazy
            return Fn(map_xs)
        return Fn(map_f)
    if k in ("reduce", "reduceSeq", "reduceSeqUnroll"):
        return Fn(lambda op: Fn(lambda init: Fn(lambda xs: _reduce(g, op, init, xs))))
    if k == "zip":
        return Fn(lambda a: Fn(lambda b: Arr(a.size, lambda i: Pair(lambda: a.elem(i), lambda: b.elem(i)), ())))
    if k == "fst":
        return Fn(lambda pr: pr.a)
    if k == "snd":
        return Fn(lambda pr: pr.b)
    if k in ("split", "asVector"):
        (n,) = p.nats
        return Fn(lambda xs: Arr(xs.size // n,
                                 lambda i: Arr(n, lambda j: xs.elem(f"(({i}) * {n} + ({j}))"), xs.inner),
                                 (n,) + xs.inner))
    if k in ("join", "asScalar"):
        def join(xs):
            m = xs.inner[0]
            return Arr(xs.size * m, lambda q: xs.elem(f"(({q}) / {m})").elem(f"(({q}) % {m})"), xs.inner[1:])
        return Fn(join)
    if k == "transpose":
        def tr(xs):
            m = xs.inner[0]
            return Arr(m, lambda j: Arr(xs.size, lambda i: xs.elem(i).elem(j), xs.inner[1:]),
                       (xs.size,) + xs.inner[1:])
        return Fn(tr)
    if k == "slide":
        sz, st = p.nats
        return Fn(lambda xs: Arr((xs.size - sz) // st + 1,
                                 lambda i: Arr(sz, lambda j: xs.elem(f"(({i}) * {st} + ({j}))"), xs.inner),
                                 (sz,) + xs.inner))
    if k == "padClamp":
        lpad, rpad = p.nats
        return Fn(lambda xs: Arr(xs.size + lpad + rpad,
                                 lambda i: xs.elem(f"min(max(({i}) - {lpad}, 0), {xs.size - 1})"), xs.inner))
    if k in ("toMem", "id"):
        return Fn(lambda v: v)
    if k == "add":
        return Fn(lambda a: Fn(lambda b: _add(a, b)))
    if k == "mult":
        return Fn(lambda a: Fn(lambda b: Prod(f"({a.code} * {b.code})", a.code, b.code)))
    raise CodegenError(f"primitive {k} is not supported by the generic compiler")


def _shape_or_scalar(v):
    if isinstance(v, Arr):
        return shape_of(v)
    if isinstance(v, Scal):
        return ()
    if isinstance(v, Pair):
        return ()
    raise CodegenError("functions cannot be array elements")


def _literal(g: Gen, value):
    if not isinstance(value, tuple):
        return Scal(_fmt(value))
    flat, shape = [], []

    def walk(v, depth):
        if isinstance(v, tuple):
            if len(shape) <= depth:
                shape.append(len(v))
            for x in v:
                walk(x, depth + 1)
        else:
            flat.append(float(v))

    walk(value, 0)
    name = g.fresh("lit")
    if not g.dry:
        g.consts.append(f"  const float {name}[{len(flat)}] = {{{', '.join(_fmt(x) for x in flat)}}};")
    return _buffer_view(g, name, tuple(shape))


def _compile(g: Gen, e, env):
    ir = S().ir
    if isinstance(e, ir.Var):
        return env[e.name]
    if isinstance(e, ir.Lit):
        return _literal(g, e.value)
    if isinstance(e, ir.Prim):
        return _prim(g, e)
    if isinstance(e, ir.Lam):
        return Fn(lambda v, e=e: _compile(g, e.body, {**env, e.param: v}))
    if isinstance(e, ir.App):
        f = _compile(g, e.fn, env)
        if not isinstance(f, Fn):
            raise CodegenError("application of a non-function")
        return f.apply(_compile(g, e.arg, env))
    raise CodegenError(f"cannot compile {e!r}")


# ----------------------------------------------------------------------------
# destination passing: where a value's elements are written

STRICT_MAP_MAX = 4096      # floats: strict (materialised) maps stay per-thread arrays
PAR_LEVELS = 2             # outermost map levels distributed over threads


@dataclass
class Out:
    """An acceptor: `lval` for a scalar destination, else `size` + `at(i)`."""
    size: int = 0
    at: Callable[[str], "Out"] = None
    lval: str = ""


def _out_buffer(buf: str, shape: tuple, base: str = "0") -> Out:
    if not shape:
        return Out(lval=f"{buf}[{base}]")
    stride = 1
    for d in shape[1:]:
        stride *= d
    return Out(shape[0], lambda i: _out_buffer(buf, shape[1:], f"({base} + ({i}) * {stride})"))


def _out_join(out: Out, m: int) -> Out:
    """X : [n/m][m] written into out : [n]."""
    return Out(out.size // m, lambda i: Out(m, lambda j: out.at(f"(({i}) * {m} + ({j}))")))


def _out_split(out: Out, n: int) -> Out:
    """X : [k*n] written into out : [k][n]."""
    return Out(out.size * n, lambda q: out.at(f"(({q}) / {n})").at(f"(({q}) % {n})"))


def _out_transpose(out: Out) -> Out:
    """X : [m][n] written into out : [n][m]."""
    m = out.at("0").size
    return Out(m, lambda i: Out(out.size, lambda j: out.at(j).at(i)))


def _write(g: Gen, v, out: Out) -> None:
    """Emit loops storing every scalar of value `v` into `out`."""
    if out.lval:
        if not isinstance(v, Scal):
            raise CodegenError("the program's result is not an array of scalars")
        g.emit(f"{out.lval} = {v.code};")
        return
    if not isinstance(v, Arr):
        raise CodegenError("the program's result is not an array of scalars")
    i = g.fresh("w")
    g.open(f"for (int {i} = 0; {i} < {v.size}; ++{i}) {{")
    _write(g, v.elem(i), out.at(i))
    g.close()


LAYOUT_PRIMS = ("join", "asScalar", "split", "asVector", "transpose", "toMem", "id")


def _layout_out(p, out: Out, x_shape: tuple) -> Out:
    """Destination for X such that writing X there writes p(X) into `out`."""
    if p.kind in ("join", "asScalar"):
        return _out_join(out, x_shape[1])
    if p.kind in ("split", "asVector"):
        return _out_split(out, p.nats[0])
    if p.kind == "transpose":
        return _out_transpose(out)
    return out


def _shape_dry(g: Gen, e, env) -> tuple:
    return g.dry_run(lambda: _shape_or_scalar(_compile(g, e, env)))


def _accept(g: Gen, e, env, out: Out, par: int) -> None:
    """Write the value of term `e` into `out`, following the term's own
    producer structure (maps become loops -- the outermost PAR_LEVELS of them
    thread indices -- layout primitives transform the destination, reduces
    run once), so no element is computed more than once."""
    ir = S().ir
    head, args = ir.spine(e)
    if isinstance(head, ir.Lam) and args:                     # (fun x => body)(a) ...
        env2 = {**env, head.param: _compile(g, args[0], env)}
        return _accept(g, ir.app(head.body, *args[1:]), env2, out, par)
    if isinstance(head, ir.Prim):
        k = head.kind
        if k in ir.MAP_KINDS and len(args) == 2:
            f, xs = args
            if isinstance(f, ir.Prim) and f.kind in LAYOUT_PRIMS:
                # map(join)(X) etc.: a per-element destination transform, no loop
                shp = _shape_dry(g, xs, env)
                return _accept(g, xs, env, Out(shp[0], lambda i: _layout_out(f, out.at(i), shp[1:])), par)
            xv = _compile(g, xs, env)
            if not isinstance(xv, Arr):
                raise CodegenError(f"{k} expects an array")
            if par > 0:
                i = f"par{len(g.par_sizes)}"
                g.par_sizes.append(xv.size)
                _accept_fn(g, f, env, xv.elem(i), out.at(i), par - 1)
            else:
                i = g.fresh("i")
                g.open(f"for (int {i} = 0; {i} < {xv.size}; ++{i}) {{")
                _accept_fn(g, f, env, xv.elem(i), out.at(i), 0)
                g.close()
            return
        if len(args) == 1 and k in LAYOUT_PRIMS:
            shp = _shape_dry(g, args[0], env)
            return _accept(g, args[0], env, _layout_out(head, out, shp), par)
    _write(g, _compile(g, e, env), out)


def _accept_fn(g: Gen, f, env, arg, out: Out, par: int) -> None:
    ir = S().ir
    if isinstance(f, ir.Lam):
        return _accept(g, f.body, {**env, f.param: arg}, out, par)
    fv = _compile(g, f, env)
    if not isinstance(fv, Fn):
        raise CodegenError("map over a non-function")
    _write(g, fv.apply(arg), out)


# ----------------------------------------------------------------------------
# kernels

@dataclass(frozen=True)
class Compiled:
    name: str
    source: str
    in_shapes: tuple       # per input: array shape
    out_shape: tuple
    threads: int = 1       # threads launched
    mode: str = ""         # "per-scalar", "register-tile TMxTN", "smem-tile ..." or "destination-passing"
    grid: tuple = ()       # explicit (x, y) grid (smem-tile mode); else 1-D over `threads`
    block: int = 128       # threads per block


def compile_term(term) -> Compiled:
    """CUDA source of `term` = fun(x0 : T0 => ... fun(xn : Tn => body)) over
    f32 arrays (see the module docstring for the two thread mappings)."""
    s = S()
    ir, tc = s.ir, s.typecheck
    try:
        ty = tc.typecheck(term)
    except tc.TypeError_ as err:
        raise CodegenError(f"ill-typed term: {err}") from None
    params = []
    t, body = ty, term
    while isinstance(t, ir.FnType):
        if not isinstance(body, ir.Lam):
            raise CodegenError("expected a lambda chain over the inputs")
        params.append((body.param, _type_shape(t.arg)))
        t, body = t.res, body.body
    out_shape = _type_shape(t)
    if not out_shape:
        raise CodegenError("the program's result is not an array of scalars")
    g = _per_scalar_kernel(body, params, out_shape)
    if g.materialised:
        # a reduce with a non-elementwise array accumulator: computing one output
        # scalar per thread would rebuild that accumulator per scalar, so write
        # the result in the term's own structure instead (destination passing)
        g = _dps_kernel(body, params, out_shape)
    else:
        g = _smem_tile(g, out_shape) or _register_tile(g, out_shape) or g
    name = "elv_generated"
    args = ", ".join([f"const float* __restrict__ in{i}" for i in range(len(params))] +
                     ["float* __restrict__ out"])
    block = g.block
    pre = [F32X2_PRELUDE] if g.grid and SMEM_F32X2 else []
    src = "\n".join(pre + [f'extern "C" __global__ void __launch_bounds__({block}) {name}({args}) {{'] + g.head +
                    g.consts + g.lines + ["}"])
    return Compiled(name, src, tuple(shp for _, shp in params), out_shape, g.threads, g.mode, g.grid, g.block)


def _inputs_env(g: Gen, params) -> dict:
    env = {}
    for idx, (p, shp) in enumerate(params):
        env[p] = _buffer_view(g, f"in{idx}", shp) if shp else Scal(f"in{idx}[0]")
    return env


def _per_scalar_kernel(body, params, out_shape) -> Gen:
    """Mode A: one thread per output scalar; lifted (elementwise) array
    reduces are folded per demanded element, so nothing is recomputed."""
    g = Gen()
    env = _inputs_env(g, params)
    total = 1
    for d in out_shape:
        total *= d
    g.head = [f"  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;",
              f"  if (t >= {total}LL) return;"]
    rem, names = "t", []
    for level, d in enumerate(out_shape):
        stride = 1
        for dd in out_shape[level + 1:]:
            stride *= dd
        g.head.append(f"  const int o{level} = (int)(({rem}) / {stride}LL);")
        g.head.append(f"  const long long r{level} = ({rem}) % {stride}LL;")
        rem = f"r{level}"
        names.append(f"o{level}")
    v = _compile(g, body, env)
    for nm in names:
        if not isinstance(v, Arr):
            raise CodegenError("the program's result is not an array of scalars")
        v = v.elem(nm)
    if not isinstance(v, Scal):
        raise CodegenError("the program's result is not an array of scalars")
    g.emit(f"out[t] = {v.code};")
    g.threads, g.mode = total, "per-scalar"
    return g


# register tiles only when enough threads remain to fill the GPU (~111 per SM)
MIN_TILE_THREADS = 16384
_DECL = re.compile(r"^float (\w+) = (.*);$")
_ASSIGN = re.compile(r"^(\w+) = (.*);$")
_FOR = re.compile(r"^for \(int (\w+) = [^;]*; \1 < [^;]*; \+\+\1\) \{$")
_OUT = re.compile(r"^out\[t\] = (.*);$")


def _register_tile(g: Gen, out_shape: tuple) -> Gen | None:
    """Mode A': a TM x TN register tile of outputs per thread (8x4, 4x4 or
    2x2, the largest that divides the result and leaves MIN_TILE_THREADS).  The per-scalar
    body of a 2-D result is a tree of counted loops (bounds independent of
    the output index) over scalar statements; every statement is replicated
    for the thread's TM x TN outputs -- rows o0 + i (O0 / TM), columns
    o1 + j (O1 / TN), so a warp's loads of a column operand stay coalesced --
    with its own copy of every local.  Each output keeps exactly the
    per-scalar operation sequence (bitwise the same results); the loads the
    tile's elements share (a row of one input, a column of the other) are
    common subexpressions of one basic block, so each is issued once for TN
    (TM) outputs instead of once per output."""
    if len(out_shape) != 2:
        return None
    O0, O1 = out_shape
    tile = None
    shapes = ((8, 4), (4, 4), (2, 2))         # measured at 1024^3: 8x4 13.8, 4x4 12.3, per-scalar 7.4 TF
    if os.environ.get("ELV_CG_TILE"):                   # tuning experiments
        shapes = (tuple(int(x) for x in os.environ["ELV_CG_TILE"].split("x")),) + shapes
    for tm, tn in shapes:
        if O0 % tm == 0 and O1 % tn == 0 and (O0 // tm) * (O1 // tn) >= MIN_TILE_THREADS:
            tile = (tm, tn)
            break
    if tile is None:
        return None
    tm, tn = tile
    locals_, body, out_expr = set(), [], None
    for line in g.lines:
        st = line.strip()
        if out_expr is not None:
            return None                                  # the output write must come last
        m = _FOR.match(st)
        if m:
            if re.search(r"\bo[01]\b", st):
                return None                              # loop bounds depend on the output index
            body.append(("for", line))
            continue
        if st == "}":
            body.append(("close", line))
            continue
        m = _DECL.match(st)
        if m:
            locals_.add(m.group(1))
            body.append(("stmt", line))
            continue
        m = _OUT.match(st)
        if m and line.startswith("  ") and not line.startswith("   "):
            out_expr = m.group(1)
            continue
        m = _ASSIGN.match(st)
        if m and m.group(1) in locals_:
            body.append(("stmt", line))
            continue
        return None
    if out_expr is None:
        return None
    names = re.compile(r"\b(" + "|".join(sorted(map(re.escape, locals_), key=len, reverse=True)) + r")\b") \
        if locals_ else None

    def inst(text, i, j):
        if names is not None:
            text = names.sub(lambda mm: f"{mm.group(1)}_{i}_{j}", text)
        text = re.sub(r"\bo0\b", f"o0_{i}", text)
        return re.sub(r"\bo1\b", f"o1_{j}", text)

    t = Gen()
    t.consts = g.consts
    q0, q1 = O0 // tm, O1 // tn
    threads = q0 * q1
    t.head = [f"  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;",
              f"  if (t >= {threads}LL) return;",
              f"  const int q0 = (int)(t / {q1}LL);",
              f"  const int q1 = (int)(t % {q1}LL);"]
    t.head += [f"  const int o0_{i} = q0 + {i * q0};" for i in range(tm)]
    t.head += [f"  const int o1_{j} = q1 + {j * q1};" for j in range(tn)]
    unroll = int(os.environ.get("ELV_CG_UNROLL", "4"))  # unroll 4: more loads in flight (+10-130 %)
    for kind, line in body:
        if kind in ("for", "close"):
            if kind == "for" and unroll > 1:
                t.lines.append(line[:len(line) - len(line.lstrip())] + f"#pragma unroll {unroll}")
            t.lines.append(line)
            continue
        indent = line[:len(line) - len(line.lstrip())]
        for i in range(tm):
            for j in range(tn):
                t.lines.append(indent + inst(line.strip(), i, j))
    for i in range(tm):
        for j in range(tn):
            t.lines.append(f"  out[(long long)o0_{i} * {O1} + o1_{j}] = {inst(out_expr, i, j)};")
    t.threads, t.mode = threads, f"register-tile {tm}x{tn}"
    return t


# ----------------------------------------------------------------------------
# Mode A'': shared-memory tiles for contractions.  When the per-scalar body of
# a 2-D result is one counted loop nest (constant trip counts, from 0) whose
# loads of an input depend on only ONE output index -- in0 on o0 (a "row"
# operand), in1 on o1 (a "column" operand), i.e. the lowered form of every
# matmul schedule -- a 256-thread block computes a 64 x 64 output tile, 4 x 4
# per thread, and stages each load site's values for CH iterations of the
# outermost loop in shared memory: rows x TL (+1 pad) for row operands,
# TL x columns for column operands (read as float4).  The per-output
# statement sequence is the per-scalar one (locals replicated per output as in
# the register-tile mode, values read from the staged copy instead of global
# memory), so the results are bitwise the per-scalar kernel's.  Host
# emulation (cpu_source) cannot run __syncthreads: this mode is GPU-only.
SMEM_TILE = True
SMEM_MIN_OUTPUTS = 1 << 16            # 256 x 256 outputs and up
SMEM_TLMAX = 32                       # staged iterations per chunk and site (x2: double-buffered)
SMEM_THREAD_TILE = (8, 4)             # outputs per thread (rows, columns)
_LOOP0 = re.compile(r"^for \(int (\w+) = 0; \1 < (\d+); \+\+\1\) \{$")


def _load_sites(text: str, inp: str):
    """(start, end, index expression) of every `inp[...]` in `text`."""
    out, pos, key = [], 0, inp + "["
    while True:
        i = text.find(key, pos)
        if i < 0:
            return out
        if i > 0 and (text[i - 1].isalnum() or text[i - 1] == "_"):
            pos = i + 1
            continue
        depth, j = 1, i + len(key)
        while depth:
            if j >= len(text):
                raise CodegenError("unbalanced index expression")
            depth += {"[": 1, "]": -1}.get(text[j], 0)
            j += 1
        out.append((i, j, text[i + len(key):j - 1]))
        pos = j


def _eval_index(expr: str, env: dict) -> int:
    """Value of a generated (non-negative) C integer index expression."""
    py = expr.replace("/", "//")
    return int(eval(py, {"__builtins__": {}}, dict(env)))   # generated text: names, ints, + * / % ( )


def _smem_tile(g: Gen, out_shape: tuple) -> Gen | None:
    if not SMEM_TILE or len(out_shape) != 2:
        return None
    O0, O1 = out_shape
    if O0 % 64 or O1 % 64 or O0 * O1 < SMEM_MIN_OUTPUTS:
        return None
    # parse the body: ("for", var, trip, children) / ("stmt", text); the output write last
    root, stack, out_expr, locals_ = [], [], None, set()
    cur = root
    for line in g.lines:
        st = line.strip()
        if out_expr is not None:
            return None
        m = _LOOP0.match(st)
        if m:
            node = ("for", m.group(1), int(m.group(2)), [])
            cur.append(node)
            stack.append(cur)
            cur = node[3]
            continue
        if st == "}":
            if not stack:
                return None
            cur = stack.pop()
            continue
        m = _OUT.match(st)
        if m and not stack:
            out_expr = m.group(1)
            continue
        m = _DECL.match(st)
        if m:
            locals_.add(m.group(1))
            cur.append(("stmt", st))
            continue
        m = _ASSIGN.match(st)
        if m and m.group(1) in locals_:
            cur.append(("stmt", st))
            continue
        return None
    if out_expr is None or stack:
        return None
    loops = [n for n in root if n[0] == "for"]
    if len(loops) != 1:
        return None
    top = loops[0]
    inputs = sorted(set(re.findall(r"\b(in\d+)\[", "\n".join(g.lines))))
    for n in root:
        if n[0] == "stmt" and any(_load_sites(n[1], i) for i in inputs):
            return None                                  # loads outside the loop nest
    if any(_load_sites(out_expr, i) for i in inputs):
        return None
    # load sites: (input, expression, enclosing inner loops) -> staging buffer
    sites, order = {}, []

    def scan(nodes, path):
        for n in nodes:
            if n[0] == "for":
                scan(n[3], path + [(n[1], n[2])])
                continue
            for inp in inputs:
                for _, _, e in _load_sites(n[1], inp):
                    r0, r1 = bool(re.search(r"\bo0\b", e)), bool(re.search(r"\bo1\b", e))
                    if r0 == r1 or re.search(r"\b(in\d+|t|q0|q1)\b", e):
                        raise CodegenError("not a contraction")
                    key = (inp, e, tuple(path))
                    if key not in sites:
                        sites[key] = {"role": "r" if r0 else "c", "inner": path}
                        order.append(key)
    try:
        scan(top[3], [])
    except CodegenError:
        return None
    if not sites or len(sites) > 4:
        return None
    v0, T0 = top[1], top[2]
    pmax = max(max(1, _prod(t for _, t in site["inner"])) for site in sites.values())
    tlmax = int(os.environ.get("ELV_CG_SMEM_TL", SMEM_TLMAX))   # tuning sweeps
    ch = 1
    for c in range(1, T0 + 1):
        if T0 % c == 0 and c * pmax <= tlmax:
            ch = c
    smem_floats = 0
    for idx, key in enumerate(order):
        site = sites[key]
        site["P"] = max(1, _prod(t for _, t in site["inner"]))
        site["TL"] = ch * site["P"]
        smem_floats += 2 * 64 * (site["TL"] + 1)
        if smem_floats * 4 > 48 * 1024 or site["TL"] > 128:
            return None                                  # static shared memory / staging registers
        site["name"] = f"sm{idx}"
        # which staging axis is contiguous in global memory (probe the index)
        loopvars = [(v0, T0)] + site["inner"]

        def env_at(tl, o, key=key, loopvars=loopvars, site=site):
            env = {"o0": o, "o1": o}
            rem = tl
            for v, t in reversed(loopvars[1:]):
                env[v] = rem % t
                rem //= t
            env[v0] = rem
            return env
        try:
            e = key[1]
            d_tl = _eval_index(e, env_at(1, 0)) - _eval_index(e, env_at(0, 0)) if site["TL"] > 1 else 0
            site["tl_fast"] = d_tl == 1
        except Exception:
            return None
    TM, TN = SMEM_THREAD_TILE
    if os.environ.get("ELV_CG_SMEM_TILE"):                 # tuning sweeps, e.g. 8x4
        TM, TN = (int(x) for x in os.environ["ELV_CG_SMEM_TILE"].split("x"))
    if TM not in (2, 4, 8) or TN not in (4, 8):
        return None
    nx, ny = 64 // TN, 64 // TM
    NT = nx * ny                                           # threads per 64 x 64 block
    t = Gen()
    t.consts = g.consts
    t.head = [f"  const int tx = threadIdx.x % {nx}, ty = threadIdx.x / {nx};",
              f"  const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;"]
    t.head += [f"  const int o0_{i} = row0 + {TM} * ty + {i};" for i in range(TM)]
    t.head += [f"  const int o1_{j} = col0 + {TN} * tx + {j};" for j in range(TN)]
    for key in order:
        site = sites[key]
        size = 64 * (site["TL"] + 1) if site["role"] == "r" else site["TL"] * 64
        site["size"] = size
        t.head.append(f"  __shared__ __align__(16) float {site['name']}[2 * {size}];")
    names = re.compile(r"\b(" + "|".join(sorted(map(re.escape, locals_), key=len, reverse=True)) + r")\b") \
        if locals_ else None

    def inst(text, i, j, loaded):
        # loads -> staged values (before any renaming: the index text names o0 / o1)
        for key in (order if loaded is not None else ()):
            inp, e, _ = key
            site = sites[key]
            if key[2] != tuple(loaded):
                continue
            rep = f"ra{site['name']}_{i}" if site["role"] == "r" else f"cb{site['name']}_{j // 4}.{'xyzw'[j % 4]}"
            text = text.replace(f"{inp}[{e}]", rep)
        if names is not None:
            text = names.sub(lambda mm: f"{mm.group(1)}_{i}_{j}", text)
        text = re.sub(r"\bo0\b", f"o0_{i}", text)
        return re.sub(r"\bo1\b", f"o1_{j}", text)

    def tl_expr(site):
        terms, stride = [], 1
        for v, tr in reversed(site["inner"]):
            terms.append(f"{v} * {stride}" if stride != 1 else v)
            stride *= tr
        terms.append(f"({v0} - {v0}_b) * {stride}")
        return " + ".join(reversed(terms))

    def emit_nodes(nodes, indent, path):
        for n in nodes:
            if n[0] == "for":
                t.lines.append(indent + "#pragma unroll")
                t.lines.append(indent + f"for (int {n[1]} = 0; {n[1]} < {n[2]}; ++{n[1]}) {{")
                emit_nodes(n[3], indent + "  ", path + [(n[1], n[2])])
                t.lines.append(indent + "}")
                continue
            st = n[1]
            used = [key for key in order if key[2] == tuple(path) and f"{key[0]}[{key[1]}]" in st]
            for key in used:
                site = sites[key]
                tl = tl_expr(site)
                if site["role"] == "r":
                    for i in range(TM):
                        t.lines.append(indent + f"const float ra{site['name']}_{i} = "
                                       f"{site['name']}[buf * {site['size']} + ({TM} * ty + {i}) * {site['TL'] + 1} + ({tl})];")
                else:
                    for h in range(TN // 4):
                        t.lines.append(indent + f"const float4 cb{site['name']}_{h} = *reinterpret_cast<const float4*>("
                                       f"&{site['name']}[buf * {site['size']} + ({tl}) * 64 + {TN} * tx + {4 * h}]);")
            for i in range(TM):
                insts = [inst(st, i, j, path) for j in range(TN)]
                t.lines.extend(indent + x for x in (_pair_f32x2(insts) if SMEM_F32X2 else insts))

    def stage_code(base_expr, store, indent):
        """Load (store=False: into registers stg<site>_<q>) or store (into the
        buffer half `buf`) the staged values of the chunk starting at
        outer-loop index `base_expr`."""
        for key in order:
            inp, e, _ = key
            site = sites[key]
            TL = site["TL"]
            total = 64 * TL
            iters = (total + NT - 1) // NT
            size = 64 * (TL + 1) if site["role"] == "r" else TL * 64
            for q in range(iters):
                t.lines.append(indent + "{")
                t.lines.append(indent + f"  const int idx = threadIdx.x + {NT * q};")
                guard = f"idx < {total}" if total % NT else None
                if site["tl_fast"]:
                    t.lines.append(indent + f"  const int tl = idx % {TL}, rr = idx / {TL};")
                else:
                    t.lines.append(indent + f"  const int tl = idx / 64, rr = idx % 64;")
                if store:
                    dst = f"rr * {TL + 1} + tl" if site["role"] == "r" else "tl * 64 + rr"
                    st = f"{site['name']}[buf * {size} + {dst}] = stg{site['name']}_{q};"
                else:
                    rem, stride = "tl", 1
                    for v, tr in reversed(site["inner"]):
                        t.lines.append(indent + f"  const int {v} = ({rem} / {stride}) % {tr};")
                        stride *= tr
                    t.lines.append(indent + f"  const int {v0} = {base_expr} + tl / {stride};")
                    o = "o0" if site["role"] == "r" else "o1"
                    base = "row0" if site["role"] == "r" else "col0"
                    ex = re.sub(rf"\b{o}\b", f"({base} + rr)", e)
                    st = f"stg{site['name']}_{q} = {inp}[{ex}];"
                t.lines.append(indent + "  " + (f"if ({guard}) " if guard else "") + st)
                t.lines.append(indent + "}")

    for n in root:
        if n is top:
            # double-buffered: the next chunk's values are loaded into registers
            # while the current chunk computes, then stored to the other half
            for key in order:
                site = sites[key]
                iters = (64 * site["TL"] + NT - 1) // NT
                t.lines.append("  float " + ", ".join(f"stg{site['name']}_{q} = 0.f" for q in range(iters)) + ";")
            t.lines.append("  int buf = 0;")
            stage_code("0", False, "  ")
            stage_code(None, True, "  ")
            t.lines.append("  __syncthreads();")
            t.lines.append(f"  for (int {v0}_b = 0; {v0}_b < {T0}; {v0}_b += {ch}, buf ^= 1) {{")
            t.lines.append(f"    const bool more = {v0}_b + {ch} < {T0};")
            t.lines.append("    if (more) {")
            stage_code(f"{v0}_b + {ch}", False, "      ")
            t.lines.append("    }")
            t.lines.append("    #pragma unroll 4")
            t.lines.append(f"    for (int {v0} = {v0}_b; {v0} < {v0}_b + {ch}; ++{v0}) {{")
            emit_nodes(top[3], "      ", [])
            t.lines.append("    }")
            t.lines.append("    if (more) {")
            t.lines.append("      buf ^= 1;")
            stage_code(None, True, "      ")
            t.lines.append("      buf ^= 1;")
            t.lines.append("    }")
            t.lines.append("    __syncthreads();")
            t.lines.append("  }")
        else:
            for i in range(TM):
                for j in range(TN):
                    t.lines.append("  " + inst(n[1], i, j, None))
    for i in range(TM):
        for j in range(TN):
            t.lines.append(f"  out[(long long)o0_{i} * {O1} + o1_{j}] = {inst(out_expr, i, j, None)};")
    t.threads = O0 * O1 // (TM * TN)
    t.grid = (O1 // 64, O0 // 64)
    t.block = NT
    t.mode = f"smem-tile {TM}x{TN} (64x64 block, {ch} x {pmax} iterations staged per chunk)"
    return t


_FMA_INST = re.compile(r"^(\w+) = fmaf\(([\w.]+), ([\w.]+), \1\);$")
_ADD_INST = re.compile(r"^(\w+) = \(\1 \+ (\w+)\);$")
SMEM_F32X2 = True                     # pair adjacent outputs' fmaf / add into sm_100 f32x2 instructions
F32X2_PRELUDE = r"""
__device__ __forceinline__ void elv_fma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  unsigned long long a, b, d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(d0), "f"(d1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}
__device__ __forceinline__ void elv_add2(float& d0, float& d1, float b0, float b1) {
  unsigned long long b, d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(d0), "f"(d1));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(d) : "l"(b));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}
"""


def _pair_f32x2(insts: list) -> list:
    """Adjacent outputs' `x = fmaf(a, b, x)` / `x = (x + y)` statements as one
    fma.rn.f32x2 / add.rn.f32x2 (each lane an IEEE fmaf / add: the same bits,
    half the FP32 issue slots -- the template kernels' FFMA2)."""
    out, j = [], 0
    while j < len(insts):
        if j + 1 < len(insts):
            m0, m1 = _FMA_INST.match(insts[j]), _FMA_INST.match(insts[j + 1])
            if m0 and m1:
                out.append(f"elv_fma2({m0.group(1)}, {m1.group(1)}, {m0.group(2)}, {m1.group(2)}, "
                           f"{m0.group(3)}, {m1.group(3)});")
                j += 2
                continue
            a0, a1 = _ADD_INST.match(insts[j]), _ADD_INST.match(insts[j + 1])
            if a0 and a1:
                out.append(f"elv_add2({a0.group(1)}, {a1.group(1)}, {a0.group(2)}, {a1.group(2)});")
                j += 2
                continue
        out.append(insts[j])
        j += 1
    return out


def _prod(xs) -> int:
    p = 1
    for x in xs:
        p *= x
    return p


def _dps_kernel(body, params, out_shape) -> Gen:
    """Mode B: destination passing; the outermost PAR_LEVELS maps are the
    thread index, small computing maps are materialised per thread."""
    g = Gen()
    g.strict_maps = True
    env = _inputs_env(g, params)
    _accept(g, body, env, _out_buffer("out", out_shape), PAR_LEVELS)
    total = 1
    for d in g.par_sizes:
        total *= d
    g.head = [f"  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;",
              f"  if (t >= {total}LL) return;"]
    stride = total
    for lvl, d in enumerate(g.par_sizes):
        stride //= d
        g.head.append(f"  const int par{lvl} = (int)((t / {stride}LL) % {d}LL);")
    g.threads, g.mode = total, "destination-passing"
    return g


def _type_shape(t) -> tuple:
    ir = S().ir
    dims = []
    while isinstance(t, ir.ArrType):
        dims.append(t.size)
        t = t.elem
    if isinstance(t, ir.VecType):
        dims.append(t.width)
        t = ir.F32
    if t != ir.F32:
        raise CodegenError(f"inputs/outputs must be f32 arrays, got {ir.format_type(t)}")
    return tuple(dims)


def cpu_source(c: Compiled) -> str:
    """The generated kernel wrapped as plain C++ (thread loop on the host), so
    tests can check code generation against the reference interpreter
    without a GPU.  Compiled with -ffp-contract=off it performs the same fp32
    operations in the same order as the NVRTC (--fmad=false, explicit fmaf) build."""
    if c.grid:
        raise CodegenError("the shared-memory tile mode needs a GPU (set codegen.SMEM_TILE = False for cpu_source)")
    n = len(c.in_shapes)
    call = ", ".join([f"ins[{i}]" for i in range(n)] + ["out"])
    return "\n".join([
        "#include <algorithm>",
        "#include <cmath>",
        "using std::min; using std::max; using std::fmaf;",
        "struct elv_dim3 { unsigned x, y, z; };",
        "static elv_dim3 blockIdx, threadIdx, blockDim;",
        "#define __global__",
        "#define __launch_bounds__(x)",
        "#define __restrict__",
        c.source,
        'extern "C" void elv_run_cpu(const float* const* ins, float* out, long long threads) {',
        "  blockDim.x = 128;",
        "  for (long long t = 0; t < threads; ++t) {",
        "    blockIdx.x = (unsigned)(t / 128); threadIdx.x = (unsigned)(t % 128);",
        f"    {c.name}({call});",
        "  }",
        "}",
    ])


# ----------------------------------------------------------------------------
# NVRTC build + driver launch

def nvrtc_cubin(compiled: Compiled) -> bytes:
    """Compile the generated source for sm_100a (no GPU needed)."""
    from cuda.bindings import nvrtc
    prog = _check(nvrtc.nvrtcCreateProgram(compiled.source.encode(), b"generated.cu", 0, [], []))
    try:
        opts = [b"--gpu-architecture=sm_100a", b"--fmad=false", b"-std=c++17", b"-default-device"]
        rc = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)[0]
        if rc != nvrtc.nvrtcResult.NVRTC_SUCCESS:
            size = _check(nvrtc.nvrtcGetProgramLogSize(prog))
            log = b" " * size
            nvrtc.nvrtcGetProgramLog(prog, log)
            raise CodegenError("NVRTC failed:\n" + log.decode(errors="replace") + "\n" + compiled.source)
        size = _check(nvrtc.nvrtcGetCUBINSize(prog))
        cubin = b" " * size
        _check(nvrtc.nvrtcGetCUBIN(prog, cubin))
        return cubin
    finally:
        nvrtc.nvrtcDestroyProgram(prog)


class Kernel:
    def __init__(self, compiled: Compiled):
        from cuda.bindings import driver
        self.c = compiled
        cubin = nvrtc_cubin(compiled)
        self.module = _check(driver.cuModuleLoadData(cubin))
        self.fn = _check(driver.cuModuleGetFunction(self.module, compiled.name.encode()))
        self.driver = driver

    def __call__(self, inputs, out, stream):
        import ctypes
        import numpy as np
        d = self.driver
        total = self.c.threads
        ptrs = [ctypes.c_void_p(t.data_ptr()) for t in list(inputs) + [out]]
        arg_ptrs = np.array([ctypes.addressof(p) for p in ptrs], dtype=np.uint64)
        if self.c.grid:
            gx, gy = self.c.grid
            _check(d.cuLaunchKernel(self.fn, gx, gy, 1, self.c.block, 1, 1, 0, d.CUstream(stream),
                                    arg_ptrs.ctypes.data, 0))
            return
        block = 128
        grid = max(1, (total + block - 1) // block)
        _check(d.cuLaunchKernel(self.fn, grid, 1, 1, block, 1, 1, 0, d.CUstream(stream),
                                arg_ptrs.ctypes.data, 0))


def _check(res):
    from cuda.bindings import driver, nvrtc
    err, *rest = res if isinstance(res, tuple) else (res,)
    if isinstance(err, nvrtc.nvrtcResult) and err != nvrtc.nvrtcResult.NVRTC_SUCCESS:
        raise CodegenError(f"NVRTC error {err}")
    if isinstance(err, driver.CUresult) and err != driver.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver error {err}")
    if not rest:
        return None
    return rest[0] if len(rest) == 1 else tuple(rest)


@functools.lru_cache(maxsize=64)
def _kernel_for_key(key: str, device_index: int, term_holder) -> Kernel:
    # a module belongs to the context it was loaded in: one Kernel per
    # (term, device), loaded while that device is current
    import torch
    with torch.cuda.device(device_index):
        torch.cuda.current_stream()              # make sure the device's primary context is current
        return Kernel(compile_term(term_holder.term))


class _Holder:
    """Hashable by the canonical print; carries the term to compile."""

    def __init__(self, key, term):
        self.key, self.term = key, term

    def __hash__(self):
        return hash(self.key)

    def __eq__(self, other):
        return isinstance(other, _Holder) and other.key == self.key


def kernel_for(term, device_index: int | None = None) -> Kernel:
    import torch
    key = S().ir.pretty(term)
    if device_index is None:
        device_index = torch.cuda.current_device()
    return _kernel_for_key(key, device_index, _Holder(key, term))


def run(term, tensors, stream=None):
    """Evaluate `term` on device tensors with a generated kernel."""
    import torch
    dev = tensors[0].device if tensors and tensors[0].is_cuda else torch.device("cuda", torch.cuda.current_device())
    k = kernel_for(term, dev.index)
    if len(tensors) != len(k.c.in_shapes):
        raise S().interp.EvalError(f"the program takes {len(k.c.in_shapes)} arguments, got {len(tensors)}")
    ins = []
    for t, shp in zip(tensors, k.c.in_shapes):
        if tuple(t.shape) != shp:
            raise S().interp.EvalError(f"argument of shape {tuple(t.shape)} where {shp} is expected")
        ins.append(t.contiguous().float())
    out = torch.empty(k.c.out_shape, device=ins[0].device, dtype=torch.float32)
    stream = stream or torch.cuda.current_stream(ins[0].device)
    with torch.cuda.device(ins[0].device):
        k(ins, out, stream.cuda_stream)
    return out
