"""Drop-in B200 backend for the reference's program evaluator.

`run(e, args)` has the signature, argument meaning and error behaviour of
`stratir.interp.run` (reference pkg/src/stratir/interp.py:157-162): it applies
the lambda-chain program `e` to `args` and returns the value.  For the terms
the seven GEMM schedules produce (see `schedules`), the evaluation runs as one
hand-written sm_100a kernel through the C ABI (include/elevate_b200.h);
anything else raises the reference's `EvalError` (interp.py:16) -- there is
no CPU fallback on this path.

Accepted argument types:
  * nested Python lists of floats (the reference's own value model; the result
    is a nested list of floats, like the reference's),
  * numpy arrays / CPU torch tensors (host buffers: copied to the GPU and back),
  * CUDA torch tensors (stay on the device; result is a CUDA tensor).

Scalars are fp32 on the device (the reference evaluates in f64,
interp.py:145-148); results match it within the sqrt(K)-scaled fp32 bound of
SURVEY.md §8(d) (see `tolerance.py`).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np
import torch

from . import _lib, dispatch
from ._ref import S

_plan_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def EvalError(msg):
    return S().interp.EvalError(msg)


def _default_tf32x3() -> bool:
    return os.environ.get("ELV_TF32X3", "0") not in ("", "0", "false", "False")


def _default_encoding() -> str:
    """Operand encoding of the tcgen05 kernel when tf32x3 is requested:
    "tf32" (the 3xTF32 split, the default: `tf32x3=True` means 3xTF32) or,
    as an explicit opt-in, "fp16" (3xFP16, power-of-two scaled fp16 planes:
    ~1.8x the throughput; rows / columns spanning more than 2^29 are
    recomputed by the range-guard fix-up; falls back to tf32 for K < 512)."""
    return os.environ.get("ELV_TC_ENCODING", "tf32")


def plan(e, arg_shapes, tf32x3: bool | None = None, tc_encoding: str | None = None) -> dispatch.KernelPlan:
    """Decode (cached per term object) and bind to the argument shapes."""
    tf32x3 = _default_tf32x3() if tf32x3 is None else tf32x3
    tc_encoding = _default_encoding() if tc_encoding is None else tc_encoding
    key = (tuple(map(tuple, arg_shapes)), bool(tf32x3), tc_encoding)
    per_term = _plan_cache.get(e)
    if per_term is None:
        per_term = {}
        try:
            _plan_cache[e] = per_term
        except TypeError:
            pass
    p = per_term.get(key)
    if p is None:
        p = dispatch.decode(e, arg_shapes, tf32x3=tf32x3, tc_encoding=tc_encoding)
        per_term[key] = p
    return p


def gemm(p: dispatch.KernelPlan, A: torch.Tensor, B: torch.Tensor,
         out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Launch the plan's kernel on device tensors (async on `stream`)."""
    lib = _lib.load()
    if not (A.is_cuda and B.is_cuda):
        raise EvalError("gemm expects CUDA tensors")
    if A.dtype != torch.float32 or B.dtype != torch.float32:
        raise EvalError("the B200 backend computes fp32 (f32 scalars, ir.py:17)")
    if A.stride(-1) != 1:
        A = A.contiguous()
    if B.stride(-1) != 1:
        B = B.contiguous()
    M, K = A.shape
    Kb, N = B.shape
    if (M, N, K) != (p.M, p.N, p.K) or Kb != K:
        raise EvalError(f"plan is for {p.M}x{p.K} . {p.K}x{p.N}, got {M}x{K} . {Kb}x{N}")
    if out is None:
        out = torch.empty((M, N), device=A.device, dtype=torch.float32)
    elif out.shape != (M, N) or out.stride(-1) != 1 or out.dtype != torch.float32:
        raise EvalError("out must be a row-major fp32 M x N tensor")
    ws_bytes = lib.elv_gemm_workspace_bytes(p.variant, M, N, K)
    ws = torch.empty(ws_bytes, device=A.device, dtype=torch.uint8) if ws_bytes else None
    cur = torch.cuda.current_stream(A.device)
    if stream is None:
        stream = cur
    elif stream != cur:
        # inputs (and any .contiguous() copies) were produced on the current
        # stream; the temporaries allocated here must not be recycled by the
        # caching allocator while `stream` still uses them
        stream.wait_stream(cur)
        for t in (A, B, out, ws):
            if t is not None:
                t.record_stream(stream)
    with torch.cuda.device(A.device):
        rc = lib.elv_gemm(p.variant, A.data_ptr(), B.data_ptr(), out.data_ptr(), M, N, K,
                          A.stride(0), B.stride(0), out.stride(0),
                          ws.data_ptr() if ws is not None else None, ws_bytes,
                          stream.cuda_stream)
    _lib.check(rc, f"elv_gemm[{p.variant_name}]")
    return out


def _one_cta_bn(M: int, N: int, sms: int) -> int:
    """N tile of the 1-CTA tensor-core kernel (csrc/tf32x3_gemm.cu one_cta_bn)."""
    best, best_cost = 256, 1e30
    for bn, eff in ((256, 1.0), (128, 0.95), (64, 0.67)):
        tiles = -(-M // 128) * -(-N // bn)
        cost = -(-tiles // sms) * bn / eff
        if cost < best_cost * 0.999:
            best, best_cost = bn, cost
    return best


def _chunk_cycles(n_mma: int, n_smem: int) -> float:
    return max(6.0 * n_mma, 5.0 * (128 + n_smem))


def pair_kernel(M: int, N: int, sms: int = 148) -> bool:
    """Whether the library runs the cta_group::2 kernel for an M x N
    tensor-core GEMM (csrc/tf32x3_gemm.cu pair_mode, defaults): at least one
    256x256 pair tile per SM, or a shorter modelled mainloop than the 1-CTA
    kernel's -- per accumulation chunk max(tensor pipe 6 n, shared memory
    5 (128 + B columns held)) cycles, times the waves."""
    pair_tiles = -(-M // 256) * -(-N // 256)
    if pair_tiles >= sms:
        return True
    pair = -(-pair_tiles // (sms // 2)) * _chunk_cycles(256, 128)
    bn = _one_cta_bn(M, N, sms)
    one = -(-(-(-M // 128) * -(-N // bn)) // sms) * _chunk_cycles(bn, bn)
    return pair < one


class GemmCall:
    """A bound kernel call with its workspace, split into the two C-ABI
    phases (elv_gemm_prepare: operand layout transform; elv_gemm_compute:
    the GEMM kernel) so callers can time or overlap them separately.
    Launches per call: prepare 0 (variants 0-3), 1 (4, 5: packB; 6: packB, or
    packA+packB fused), 2 (7: guard-flag zeroing, fused hi/lo split of A and
    B), 3 (8: column-maxima zeroing, [A rows | B maxima], B split) -- each
    prepare PDL-chained; compute 1, or 2 for the tensor-core variants when the
    range-guard fix-up runs as its own launch (see count_launches)."""

    PREPARE_LAUNCHES = {0: 0, 1: 0, 2: 0, 3: 0, 4: 1, 5: 1, 6: 1, 7: 2, 8: 3}

    @classmethod
    def count_launches(cls, p) -> int:
        """Kernel launches of one call (the library's defaults): the
        tensor-core variants fold the range-guard fix-up into the 1-CTA GEMM
        (the small problems `pair_kernel` leaves to it); the prepare counts
        as PREPARE_LAUNCHES; K < 512 runs variant 8 as 7."""
        if p.variant not in (7, 8):
            return cls.PREPARE_LAUNCHES[p.variant] + 1
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count \
            if torch.cuda.is_available() else 148
        # the library's own rule (elv_tc_kernel_choice); pair_kernel mirrors it
        pair = _lib.load().elv_tc_kernel_choice(max(p.M, 1), max(p.N, 1), sms, None) == 1
        compute = 2 if pair else 1
        if p.variant == 8 and p.K >= 512:
            return cls.PREPARE_LAUNCHES[8] + compute
        return cls.PREPARE_LAUNCHES[7] + compute

    def __init__(self, p: dispatch.KernelPlan, A, B, C, stream=None):
        self.lib = _lib.load()
        self.p, self.A, self.B, self.C = p, A, B, C
        self.stream = stream or torch.cuda.current_stream(A.device)
        self.ws_bytes = self.lib.elv_gemm_workspace_bytes(p.variant, p.M, p.N, p.K)
        self.ws = (torch.empty(self.ws_bytes, device=A.device, dtype=torch.uint8)
                   if self.ws_bytes else None)
        self.launches = self.count_launches(p)
        # the buffers are fixed for the object's lifetime: build the C-ABI
        # argument tuples once (saves 1.5-3 us of host time per 1024^3 call,
        # 5-8 % of a single 3xTF32 / SIMT call; profiles/r1/small/gemmcall_args.jsonl)
        ws = (self.ws.data_ptr() if self.ws is not None else None, self.ws_bytes, self.stream.cuda_stream)
        self._prep_args = (p.variant, A.data_ptr(), B.data_ptr(), p.M, p.N, p.K, A.stride(0), B.stride(0), *ws)
        self._comp_args = (p.variant, A.data_ptr(), B.data_ptr(), C.data_ptr(), p.M, p.N, p.K, A.stride(0),
                           B.stride(0), C.stride(0), *ws)
        self._prep_fn, self._comp_fn = self.lib.elv_gemm_prepare, self.lib.elv_gemm_compute
        self._dev = A.device.index

    def _on_device(self, fn, args, what):
        # the C ABI launches into the current device's context: switch only
        # when the operands live elsewhere (a device guard costs ~2 us per use)
        if torch.cuda.current_device() != self._dev:
            with torch.cuda.device(self._dev):
                rc = fn(*args)
        else:
            rc = fn(*args)
        if rc:
            _lib.check(rc, what)

    def prepare(self):
        self._on_device(self._prep_fn, self._prep_args, "elv_gemm_prepare")

    def compute(self):
        self._on_device(self._comp_fn, self._comp_args, "elv_gemm_compute")

    def __call__(self):
        self.prepare()
        self.compute()
        return self.C

    def graph(self) -> "torch.cuda.CUDAGraph":
        """The call's launches (prepare + compute: memsets, kernels, PDL
        edges) captured once into a CUDA graph on a side stream; `replay()`
        re-runs them as one graph launch on the current stream -- the host
        launch overhead of a small call (several ctypes calls and launches)
        is paid once.  Same kernels, same arguments, same bits."""
        if getattr(self, "_graph", None) is None:
            self()                                      # first launches outside capture (attributes, modules)
            torch.cuda.synchronize(self.A.device)
            cap = torch.cuda.Stream(self.A.device)
            ws = (self.ws.data_ptr() if self.ws is not None else None, self.ws_bytes, cap.cuda_stream)
            p, A, B, C = self.p, self.A, self.B, self.C
            prep = (p.variant, A.data_ptr(), B.data_ptr(), p.M, p.N, p.K, A.stride(0), B.stride(0), *ws)
            comp = (p.variant, A.data_ptr(), B.data_ptr(), C.data_ptr(), p.M, p.N, p.K, A.stride(0),
                    B.stride(0), C.stride(0), *ws)
            g = torch.cuda.CUDAGraph()
            cap.wait_stream(torch.cuda.current_stream(self.A.device))
            with torch.cuda.device(self._dev), torch.cuda.graph(g, stream=cap):
                _lib.check(self._prep_fn(*prep), "elv_gemm_prepare (graph capture)")
                _lib.check(self._comp_fn(*comp), "elv_gemm_compute (graph capture)")
            self._graph = g
        return self._graph


def run_tensor(e, A: torch.Tensor, B: torch.Tensor, out=None, stream=None,
               tf32x3: bool | None = None, tc_encoding: str | None = None) -> torch.Tensor:
    """Tensor-returning variant of `run`: device in, device out, async."""
    p = plan(e, [tuple(A.shape), tuple(B.shape)], tf32x3, tc_encoding)
    return gemm(p, A, B, out=out, stream=stream)


def _as_host_f32(x):
    if isinstance(x, list):
        try:
            return torch.tensor(x, dtype=torch.float32)
        except (TypeError, ValueError) as err:
            raise EvalError(f"map expects an array: {err}") from None
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if isinstance(x, torch.Tensor):
        return x
    raise EvalError(f"map expects an array, got {type(x).__name__}")


class HostPipeline:
    """Host-resident A, B -> host C with the transfers overlapped: a thin
    binding of the C-ABI host pipeline `elv_gemm_host` (csrc/host_pipeline.cu).

    The output is cut into R x Nc tiles (or, for the tensor-core variants on
    large outputs, A and B arrive in strips and each landed strip is
    multiplied against the other operand's resident prefix); operands cross
    PCIe on the library's H2D stream in first-use order, each block is
    prepared (packB / tf32 / fp16 split) and multiplied on the compute stream
    as soon as its operands land, and goes back on the D2H stream as soon as
    it is written (PCIe is full duplex).  Blocks of C are independent (the
    mapPar axis) and each block's per-element arithmetic is the single-launch
    kernel's, so the result is bit-identical to `gemm`.  The device workspace
    (A, B, C and the prepared operands) is torch-owned and cached here."""

    def __init__(self, p: dispatch.KernelPlan, device):
        self.lib = _lib.load()
        self.p, self.device = p, device
        self.ws_bytes = self.lib.elv_gemm_host_workspace_bytes(p.variant, p.M, p.N, p.K)
        self.ws = torch.empty(self.ws_bytes, device=device, dtype=torch.uint8)
        r, c = ctypes.c_int(), ctypes.c_int()
        _lib.check(self.lib.elv_gemm_host_tiles(p.variant, p.M, p.N, p.K, ctypes.byref(r),
                                                ctypes.byref(c)), "elv_gemm_host_tiles")
        self.tile = (r.value, c.value)
        # one call at a time per workspace: concurrent callers (threads on
        # other streams) would otherwise share A/B/C staging buffers
        self._lock = threading.Lock()
        self._done = None           # event: the previous call's work has drained

    def __call__(self, A_h: torch.Tensor, B_h: torch.Tensor, out_h: torch.Tensor,
                 sync: bool = True) -> torch.Tensor:
        p = self.p
        for t, shape in ((A_h, (p.M, p.K)), (B_h, (p.K, p.N)), (out_h, (p.M, p.N))):
            if t.is_cuda or t.dtype != torch.float32 or tuple(t.shape) != shape or t.stride(-1) != 1:
                raise EvalError(f"host pipeline expects row-major fp32 host matrices {shape}")
        st = torch.cuda.current_stream(self.device)
        with self._lock:
            if self._done is not None:
                st.wait_event(self._done)     # previous call (maybe another stream) done with the workspace
            with torch.cuda.device(self.device):
                rc = self.lib.elv_gemm_host(p.variant, A_h.data_ptr(), B_h.data_ptr(), out_h.data_ptr(),
                                            p.M, p.N, p.K, A_h.stride(0), B_h.stride(0), out_h.stride(0),
                                            self.ws.data_ptr(), self.ws_bytes, st.cuda_stream)
            _lib.check(rc, f"elv_gemm_host[{p.variant_name}]")
            self._done = torch.cuda.Event()
            self._done.record(st)
        if sync:
            st.synchronize()
        return out_h


_host_pipes: dict = {}


def host_pipeline(p: dispatch.KernelPlan, device) -> HostPipeline:
    """One cached HostPipeline (and its device workspace) per plan and device."""
    key = (p.variant, p.M, p.N, p.K, str(device))
    hp = _host_pipes.get(key)
    if hp is None:
        if len(_host_pipes) >= 4:
            _host_pipes.clear()
        hp = _host_pipes[key] = HostPipeline(p, device)
    return hp


_PIPELINE_MIN_BYTES = 64 << 20


def _run_binomial(e, img, device=None):
    """The one-argument programs: the binomial-filter schedules (binomial.py)."""
    from . import binomial
    variant, H, W = binomial.decode(e)
    kind = type(img)
    t = _as_host_f32(img)
    if t.dim() != 2 or tuple(t.shape) != (H, W):
        raise EvalError(f"the term is typed for a {H}x{W} image, got {tuple(t.shape)}")
    if device is None:
        device = t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())
    src = t.to(device, torch.float32).contiguous()
    out = torch.empty_like(src)
    binomial.launch(variant, src, out)
    if kind is list:
        return out.double().cpu().tolist()
    if kind is np.ndarray:
        return out.cpu().numpy()
    return out if t.is_cuda else out.cpu()


def _no_template(err) -> bool:
    return str(err).startswith("no B200 kernel for term")


def _run_generic(e, args, device=None):
    """Programs the template dispatch does not recognise: one generated
    kernel per term (codegen.py, the GPU analogue of SPEC's codegen-c)."""
    from . import codegen
    kinds = [type(a) for a in args]
    ts = [_as_host_f32(a) for a in args]
    if device is None:
        cuda_in = [t for t in ts if t.is_cuda]
        device = cuda_in[0].device if cuda_in else torch.device("cuda", torch.cuda.current_device())
    try:
        out = codegen.run(e, [t.to(device, torch.float32) for t in ts])
    except codegen.CodegenError as err:
        raise EvalError(f"no B200 kernel for term: {err}") from None
    if kinds and kinds[0] is list:
        return out.double().cpu().tolist()
    if kinds and kinds[0] is np.ndarray:
        return out.cpu().numpy()
    return out if (ts and ts[0].is_cuda) else out.cpu()


def run(e, args: list, *, device=None, tf32x3: bool | None = None, out=None, tc_encoding: str | None = None):
    """Evaluate the program `e` applied to `args` on a B200.

    Mirrors stratir.interp.run (interp.py:157-162).  The seven GEMM schedules
    and the four binomial schedules run their hand-written kernels (template
    dispatch); any other well-typed program over the primitive vocabulary runs
    a generated kernel (codegen.py).  Host inputs are copied to the GPU and
    the result comes back in the caller's representation (nested lists for
    lists, numpy for numpy, tensors for tensors).  `out` (optional, GEMM
    path) is a preallocated M x N fp32 tensor -- e.g. pinned host memory --
    the result is written into and returned.  Large host-resident GEMMs go
    through `HostPipeline` (transfers overlapped with the kernel)."""
    try:
        return _run_template(e, args, device=device, tf32x3=tf32x3, out=out, tc_encoding=tc_encoding)
    except S().interp.EvalError as err:
        if not _no_template(err):
            raise
        return _run_generic(e, args, device)


def _operand_shape(x):
    """(rows, cols) of a matrix operand; cols is None for an empty list (no
    row to read it from); None when x is not a 2-D operand."""
    if isinstance(x, list):
        if not x:
            return 0, None
        if not isinstance(x[0], list):
            return None
        return len(x), len(x[0])
    if isinstance(x, (np.ndarray, torch.Tensor)) and x.ndim == 2:
        return int(x.shape[0]), int(x.shape[1])
    return None


def _truncate_ragged(b):
    """Every schedule reads B through `transpose`, which is `zip(*m)` in the
    reference (interp.py:115-120): rows of unequal length are cut to the
    shortest.  Mirror that for nested-list B (ragged A raises EvalError on
    both sides: zip of unequal lengths)."""
    if isinstance(b, list) and b and all(isinstance(r, list) for r in b):
        n = min(len(r) for r in b)
        if any(len(r) != n for r in b):
            return [r[:n] for r in b]
    return b


def _empty_gemm(e, args, out):
    """Zero-extent GEMMs, answered from the shapes alone -- there is no
    arithmetic to run -- with the reference interpreter's outcome:
      * no rows in A: `map` over [] is [] (interp.py:80-83), whatever B is;
      * rows, but B has no rows (K = 0): `transpose` of an empty array
        raises EvalError (interp.py:115-120);
      * rows, K > 0, no columns in B: the baseline schedule maps over the
        empty transpose -> M empty rows; the tiled schedules transpose an
        empty column tile and raise the same EvalError.
    Returns None when no extent is zero (the kernel path runs)."""
    sa, sb = _operand_shape(args[0]), _operand_shape(args[1])
    if sa is None or sb is None:
        return None
    (M, K), (K2, N) = sa, sb
    if M and K2 and N:
        return None
    name = dispatch.decode(e).schedule        # EvalError unless e is one of the seven GEMM schedules
    if M and not K2:
        raise EvalError("transpose of empty array")
    if M and name != "baseline":
        raise EvalError("transpose of empty array")
    n = N or 0
    if isinstance(args[0], list):
        return [[] for _ in range(M)]
    if out is not None:
        return out
    if isinstance(args[0], np.ndarray):
        return np.zeros((M, n), dtype=np.float32)
    return torch.empty((M, n), dtype=torch.float32, device=args[0].device)


def _run_template(e, args: list, *, device=None, tf32x3: bool | None = None, out=None,
                  tc_encoding: str | None = None):
    if len(args) == 1:
        return _run_binomial(e, args[0], device)
    if len(args) != 2:
        raise EvalError(f"no B200 kernel for term: {len(args)}-argument program")
    kinds = [type(a) for a in args]
    args = [args[0], _truncate_ragged(args[1])]
    empty = _empty_gemm(e, args, out)
    if empty is not None:
        return empty
    ts = [_as_host_f32(a) for a in args]
    for t in ts:
        if t.dim() != 2:
            # not matrix operands: a program that is no GEMM schedule (vector
            # add / dot, ...) goes to the generic compiler ("no B200 kernel"),
            # a GEMM schedule fails like the reference's map over scalars
            dispatch.term_shape(e)
            raise EvalError("map expects an array of arrays")
    p = plan(e, [tuple(t.shape) for t in ts], tf32x3, tc_encoding)
    if device is None:
        device = ts[0].device if ts[0].is_cuda else torch.device("cuda", torch.cuda.current_device())
    on_host = not ts[0].is_cuda
    if (on_host and not ts[1].is_cuda and p.M >= 256
            and 4 * (p.M * p.K + p.M * p.N) >= _PIPELINE_MIN_BYTES
            and (out is None or not out.is_cuda)):
        A_h = ts[0].contiguous().float()
        B_h = ts[1].contiguous().float()
        dst = out if out is not None else torch.empty((p.M, p.N), dtype=torch.float32,
                                                      pin_memory=A_h.is_pinned())
        with torch.cuda.device(device):
            host_pipeline(p, device)(A_h, B_h, dst)
        if kinds[0] is list:
            return dst.double().tolist()
        if kinds[0] is np.ndarray:
            return dst.numpy()
        return dst
    A = ts[0].to(device, torch.float32, non_blocking=True)
    B = ts[1].to(device, torch.float32, non_blocking=True)
    if out is not None and out.is_cuda:
        return gemm(p, A, B, out=out)
    C = gemm(p, A, B)
    if out is not None:
        out.copy_(C, non_blocking=out.is_pinned())
        torch.cuda.current_stream(C.device).synchronize()
        return out
    if kinds[0] is list:
        return C.double().cpu().tolist()
    if kinds[0] is np.ndarray:
        return C.cpu().numpy()
    if on_host:
        return C.cpu()
    return C
