"""Counter-based synthetic inputs, bit-identical on host (numpy) and device.

X[i] = (m - 2^23) / 2^23 with m = splitmix64((seed << 48) ^ (tensor_id << 40)
^ (offset + i)) >> 40, i.e. U(-1, 1) on a 24-bit grid: every value is exact
in fp32 and `tolist()` feeds the f64 reference interpreter without rounding
(SURVEY.md §8(d)).  The device twin is `elv_fill_uniform` (csrc/elv_api.cu),
so 1 GiB shards are generated on the GPU and any row slice is regenerated on
the host for the oracle.  Tensor ids: A = 0, B = 1.
"""

from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(n: int, seed: int = 0, tensor_id: int = 0, offset: int = 0) -> np.ndarray:
    key = np.uint64(((seed << 48) ^ (tensor_id << 40)) & 0xFFFFFFFFFFFFFFFF)
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    h = _splitmix64(key ^ idx)
    m = (h >> np.uint64(40)).astype(np.int64)
    return ((m - (1 << 23)).astype(np.float32) * np.float32(1.0 / (1 << 23))).astype(np.float32)


def matrix(rows: int, cols: int, seed: int = 0, tensor_id: int = 0,
           row0: int = 0, ld: int | None = None) -> np.ndarray:
    """rows x cols block starting at row `row0` of a matrix with `ld` columns."""
    ld = cols if ld is None else ld
    if ld == cols:
        return uniform(rows * cols, seed, tensor_id, row0 * ld).reshape(rows, cols)
    out = np.empty((rows, cols), np.float32)
    for r in range(rows):
        out[r] = uniform(cols, seed, tensor_id, (row0 + r) * ld)
    return out


def fill_device(t, seed: int = 0, tensor_id: int = 0, offset: int = 0) -> None:
    """Fill a contiguous float32 CUDA tensor in place with the same values."""
    import torch
    from . import _lib
    assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
    lib = _lib.load()
    stream = torch.cuda.current_stream(t.device).cuda_stream
    _lib.check(lib.elv_fill_uniform(t.data_ptr(), t.numel(), seed, tensor_id, offset, stream),
               "elv_fill_uniform")
