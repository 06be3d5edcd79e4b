"""ctypes binding of libelevate_b200.so (the C ABI in include/elevate_b200.h).

There is no fallback: if the library is missing or fails to load, every
entry point raises.  Build it with `python -m paper_2002_02268_b200.build`.
"""

from __future__ import annotations

import ctypes
import os

from ._ref import S

LIB_PATH = os.environ.get("ELV_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                   "libelevate_b200.so")

ELV_OK, ELV_EINVAL, ELV_EVARIANT, ELV_ECUDA, ELV_ENCCL, ELV_EWORKSPACE = 0, -1, -2, -3, -4, -5

# every symbol include/elevate_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "elv_gemm", "elv_gemm_prepare", "elv_gemm_compute", "elv_gemm_workspace_bytes", "elv_gemm_prepacked", "elv_pack_b",
    "elv_pack_b_bytes", "elv_split_tf32", "elv_fill_uniform", "elv_nccl_init",
    "elv_nccl_destroy", "elv_gemm_rowshard", "elv_last_error", "elv_abi_version",
    "elv_variant_name", "elv_tf32x3_a_planes_bytes", "elv_tf32x3_b_planes_bytes",
    "elv_tf32x3_split_a", "elv_tf32x3_split_b", "elv_tf32x3_split_b_packed",
    "elv_tf32x3_gemm_planes", "elv_tc_kernel_choice", "elv_tf32x3_fused_ok", "elv_tf32x3_gemm_fused", "elv_tf32x3_gemm_fused_a",
    "elv_binomial", "elv_binomial_variant_name",
    "elv_gemm_host", "elv_gemm_host_workspace_bytes", "elv_gemm_host_tiles", "elv_gemm_host_trace", "elv_copy2d",
    "elv_fp16x3_a_planes_bytes", "elv_fp16x3_b_planes_bytes", "elv_fp16x3_applicable", "elv_fp16x3_split_a",
    "elv_fp16x3_split_b", "elv_fp16x3_gemm_planes", "elv_fp16x3_split_b_packed", "elv_tc_fixup",
    "elv_gemm_rowshard_workspace_bytes", "elv_gemm_rowshard_pipelined",
)

_lib = None

c_int, c_ll, c_ull, c_size, c_vp, c_uint = (ctypes.c_int, ctypes.c_longlong, ctypes.c_ulonglong,
                                            ctypes.c_size_t, ctypes.c_void_p, ctypes.c_uint)


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: the CUDA backend is not built "
                           "(python -m paper_2002_02268_b200.build); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "elv_gemm": (c_int, [c_int, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_int,
                             c_vp, c_size, c_vp]),
        "elv_gemm_prepare": (c_int, [c_int, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int,
                                     c_vp, c_size, c_vp]),
        "elv_gemm_compute": (c_int, [c_int, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int,
                                     c_int, c_vp, c_size, c_vp]),
        "elv_gemm_workspace_bytes": (c_size, [c_int, c_int, c_int, c_int]),
        "elv_gemm_prepacked": (c_int, [c_int, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_vp]),
        "elv_pack_b": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp]),
        "elv_pack_b_bytes": (c_size, [c_int, c_int]),
        "elv_split_tf32": (c_int, [c_vp, c_vp, c_vp, c_ll, c_vp]),
        "elv_fill_uniform": (c_int, [c_vp, c_ll, c_ull, c_uint, c_ll, c_vp]),
        "elv_nccl_init": (c_int, [c_int, ctypes.POINTER(c_int)]),
        "elv_nccl_destroy": (c_int, []),
        "elv_gemm_rowshard": (c_int, [c_int, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_vp),
                                      ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                                      ctypes.POINTER(c_int), c_int, c_int, ctypes.POINTER(c_vp)]),
        "elv_gemm_rowshard_workspace_bytes": (c_size, [c_int, c_int, c_int, c_int, c_int]),
        "elv_gemm_rowshard_pipelined": (c_int, [c_int, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_vp), c_vp,
                                                ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_int),
                                                c_int, c_int, c_int, ctypes.POINTER(c_vp), c_size,
                                                ctypes.POINTER(c_vp)]),
        "elv_tf32x3_a_planes_bytes": (c_size, [c_int, c_int]),
        "elv_tf32x3_b_planes_bytes": (c_size, [c_int, c_int]),
        "elv_tf32x3_split_a": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp]),
        "elv_tf32x3_split_b": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp]),
        "elv_tf32x3_split_b_packed": (c_int, [c_vp, c_int, c_int, c_vp, c_vp]),
        "elv_tf32x3_gemm_planes": (c_int, [c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp]),
        "elv_tf32x3_fused_ok": (c_int, [c_vp, c_int, c_vp, c_int, c_int, c_int]),
        "elv_tc_kernel_choice": (c_int, [c_int, c_int, c_int, c_vp]),
        "elv_tf32x3_gemm_fused": (c_int, [c_vp, c_int, c_vp, c_int, c_vp, c_int, c_int, c_int, c_int, c_vp, c_vp]),
        "elv_tf32x3_gemm_fused_a": (c_int, [c_vp, c_int, c_vp, c_vp, c_int, c_vp, c_int, c_int, c_int, c_int, c_vp,
                                            c_vp]),
        "elv_gemm_host": (c_int, [c_int, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_int,
                                  c_vp, c_size, c_vp]),
        "elv_gemm_host_workspace_bytes": (c_size, [c_int, c_int, c_int, c_int]),
        "elv_gemm_host_tiles": (c_int, [c_int, c_int, c_int, c_int, ctypes.POINTER(c_int),
                                        ctypes.POINTER(c_int)]),
        "elv_gemm_host_trace": (c_int, [c_vp, c_int]),
        "elv_copy2d": (c_int, [c_vp, c_size, c_vp, c_size, c_size, c_size, c_int, c_vp]),
        "elv_fp16x3_a_planes_bytes": (c_size, [c_int, c_int]),
        "elv_fp16x3_b_planes_bytes": (c_size, [c_int, c_int]),
        "elv_fp16x3_applicable": (c_int, [c_int, c_int, c_int]),
        "elv_fp16x3_split_a": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp]),
        "elv_fp16x3_split_b": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp]),
        "elv_fp16x3_gemm_planes": (c_int, [c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp]),
        "elv_fp16x3_split_b_packed": (c_int, [c_vp, c_int, c_int, c_vp, c_vp]),
        "elv_tc_fixup": (c_int, [c_int, c_vp, c_vp, c_vp, c_int, c_vp, c_int, c_int, c_vp, c_int, c_int, c_int,
                                 c_int, c_vp]),
        "elv_binomial": (c_int, [c_int, c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp]),
        "elv_binomial_variant_name": (ctypes.c_char_p, [c_int]),
        "elv_last_error": (ctypes.c_char_p, []),
        "elv_abi_version": (c_int, []),
        "elv_variant_name": (ctypes.c_char_p, [c_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.elv_abi_version() != 1:
        raise RuntimeError("libelevate_b200 ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map C-ABI status codes onto the reference's error conventions."""
    if rc == ELV_OK:
        return
    msg = (_lib.elv_last_error() or b"").decode(errors="replace")
    if rc in (ELV_EINVAL, ELV_EVARIANT, ELV_EWORKSPACE):
        raise S().interp.EvalError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({rc}): {msg}")
