"""CPU: the C-ABI library loads, exports every declared symbol, and its
argument checking follows the reference's error conventions -- without
launching anything (no GPU here)."""

import ctypes
import os
import re

import pytest

from paper_2002_02268_b200 import _lib
from paper_2002_02268_b200._ref import S

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "elevate_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(elv_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_binding_table():
    assert set(declared_symbols()) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_abi_metadata():
    lib = _lib.load()
    assert lib.elv_abi_version() == 1
    names = [lib.elv_variant_name(v).decode() for v in range(8)]
    assert names == ["baseline", "blocking", "vectorized", "loopPerm", "arrayPacking",
                     "cacheBlocks", "parallel", "parallel_tf32x3"]
    assert lib.elv_variant_name(99) == b"unknown"


def test_workspace_sizes():
    lib = _lib.load()
    for v in range(4):
        assert lib.elv_gemm_workspace_bytes(v, 1024, 1024, 1024) == 0
    # packedB: ceil(N/256)*256 columns x K rows of fp32
    for v in (4, 5):
        assert lib.elv_gemm_workspace_bytes(v, 100, 1000, 33) == 1024 * 33 * 4
    # parallel: + packedA (ceil(M/128)*128 rows x K) for small problems (64x64-tile
    # kernel) and large ones (cp.async 128x256 kernel)
    assert lib.elv_gemm_workspace_bytes(6, 100, 1000, 33) == 1024 * 33 * 4 + 128 * 33 * 4
    assert lib.elv_pack_b_bytes(33, 1000) == 1024 * 33 * 4
    # 3xTF32: hi/lo planes of A (M x Kp) and B^T (N x Kp), Kp = K rounded to 32, each
    # with its range-guard flags (rows u32, 128 B-rounded), + the workspace's
    # contiguous flag tail (M + N u32) and alignment slack
    up = lambda x: (x + 127) // 128 * 128  # noqa: E731
    planes = (2 * 100 * 32 + 2 * 200 * 32) * 4 + 256 + up(100 * 4) + up(200 * 4)
    assert lib.elv_gemm_workspace_bytes(7, 100, 200, 30) == planes + 128 + up(300 * 4)
    assert lib.elv_gemm_workspace_bytes(0, 0, 5, 5) == 0


def test_argument_errors_map_to_eval_error():
    lib = _lib.load()
    EvalError = S().interp.EvalError
    rc = lib.elv_gemm(0, None, None, None, 4, 4, 4, 4, 4, 4, None, 0, None)
    assert rc == _lib.ELV_EINVAL
    assert b"null" in lib.elv_last_error()
    with pytest.raises(EvalError):
        _lib.check(rc, "elv_gemm")
    fake = ctypes.c_void_p(16)   # never dereferenced: rejected before any launch
    assert lib.elv_gemm(0, fake, fake, fake, 0, 4, 4, 4, 4, 4, None, 0, None) == _lib.ELV_EINVAL
    assert lib.elv_gemm(0, fake, fake, fake, 4, 4, 4, 2, 4, 4, None, 0, None) == _lib.ELV_EINVAL
    assert lib.elv_gemm(42, fake, fake, fake, 4, 4, 4, 4, 4, 4, None, 0, None) == _lib.ELV_EVARIANT
    assert lib.elv_gemm(6, fake, fake, fake, 4, 4, 4, 4, 4, 4, None, 0, None) == _lib.ELV_EWORKSPACE
    assert lib.elv_pack_b(fake, fake, 4, 4, 4, 16, None) == _lib.ELV_EINVAL
    assert lib.elv_gemm_prepacked(2, fake, fake, fake, 4, 4, 4, 4, 4, None) == _lib.ELV_EVARIANT
    assert lib.elv_gemm_rowshard(6, 1, None, None, None, None, None, None, 4, 4, None) == _lib.ELV_EINVAL
    assert lib.elv_split_tf32(fake, fake, fake, -1, None) == _lib.ELV_EINVAL
    assert lib.elv_fill_uniform(None, 4, 0, 0, 0, None) == _lib.ELV_EINVAL


def test_runtime_errors_map_to_runtime_error():
    _lib.load()
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ELV_ECUDA, "x")
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ELV_ENCCL, "x")


def test_kernel_choice_matches_the_python_mirror():
    """elv_tc_kernel_choice (the library's default pair / 1-CTA rule; no
    device work) agrees with interp.pair_kernel / _one_cta_bn, which
    GemmCall.count_launches (the bench's gpu_launches claim) uses, over a
    sweep of output shapes and SM counts."""
    import ctypes
    from paper_2002_02268_b200 import _lib, interp
    lib = _lib.load()
    bn = ctypes.c_int(0)
    shapes = [(m, n) for m in (1, 100, 128, 257, 640, 1000, 1024, 1536, 2048, 2304, 3072, 4096, 8192, 32768)
              for n in (1, 64, 256, 513, 1031, 1024, 2048, 2304, 4096, 32768)]
    for sms in (148, 132, 160):
        for m, n in shapes:
            pair = lib.elv_tc_kernel_choice(m, n, sms, ctypes.byref(bn))
            assert pair == int(interp.pair_kernel(m, n, sms)), (m, n, sms)
            assert bn.value == interp._one_cta_bn(m, n, sms), (m, n, sms)
    assert lib.elv_tc_kernel_choice(0, 10, 148, None) == _lib.ELV_EINVAL
