"""Row-sharded multi-GPU evaluation of the parallel schedule (one process/GPU).

The parallel schedule's outer `mapPar` runs over `split(32)(a)` -- the row
blocks of A and C (the TVM `s[C].parallel(xo)` axis, reference PAPER.md:80;
`mapPar` evaluates each row independently, interp.py:80-83).  That axis is the
shard axis: rank r owns rows [row0_r, row0_r + rows_r) of A and C and
computes them with the single-GPU kernel.  The only exchange is B, which
starts on rank 0 (the caller's second argument) and is broadcast with NCCL
over NVLink before the kernel reads it.  C stays sharded.

No reduction collective exists on this path (rows are independent), so none
is added.  Host-side logic here is covered on CPU with gloo (world_size 2) in
tests/test_distributed.py via an injected compute function; the product path
always computes with `interp.gemm` (the CUDA kernels).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

ROW_ALIGN = 128     # the kernels' CTA row tile; shards are multiples of it


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    row0: int
    rows: int


def shard_rows(M: int, world: int, rank: int, align: int = ROW_ALIGN) -> Shard:
    """Contiguous, tile-aligned row blocks; the last ranks absorb the tail.

    Every row lands on exactly one rank; all shards but the last are a
    multiple of `align` so per-row arithmetic (tile position inside the
    kernel) matches the 1-GPU run."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    blocks = (M + align - 1) // align
    base, extra = divmod(blocks, world)
    b0 = rank * base + min(rank, extra)
    nb = base + (1 if rank < extra else 0)
    row0 = min(b0 * align, M)
    rows = max(0, min((b0 + nb) * align, M) - row0)
    return Shard(rank, world, row0, rows)


class RowShardGemm:
    """C_shard = A_shard . B on every rank, B broadcast from `src`.

    `compute(A_shard, B, C_shard)` defaults to the CUDA kernel of `plan`;
    tests inject a CPU function to exercise the sharding logic with gloo.
    """

    def __init__(self, plan=None, group=None, src: int = 0, compute=None, stream=None):
        self.plan = plan
        self.group = group
        self.src = src
        self.stream = stream
        if compute is None:
            from . import interp

            def compute(A, B, C):
                return interp.gemm(plan, A, B, out=C, stream=stream)
        self.compute = compute

    def broadcast_b(self, B: torch.Tensor) -> torch.Tensor:
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.broadcast(B, src=self.src, group=self.group)
        return B

    def step(self, A_shard: torch.Tensor, B: torch.Tensor, C_shard: torch.Tensor) -> torch.Tensor:
        self.broadcast_b(B)
        if A_shard.shape[0] == 0:
            return C_shard
        return self.compute(A_shard, B, C_shard)


def gather_rows(C_shard: torch.Tensor, M: int, group=None, align: int = ROW_ALIGN) -> torch.Tensor:
    """Optional: assemble the full C on every rank (not on the timed path).
    Shards are padded to the largest shard for the equal-size all_gather."""
    world = dist.get_world_size(group)
    N = C_shard.shape[1]
    shards = [shard_rows(M, world, r, align) for r in range(world)]
    mx = max(s.rows for s in shards)
    buf = torch.zeros((mx, N), dtype=C_shard.dtype, device=C_shard.device)
    buf[:C_shard.shape[0]] = C_shard
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:s.rows] for p, s in zip(parts, shards)], 0)
