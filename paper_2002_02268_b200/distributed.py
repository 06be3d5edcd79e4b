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


def column_chunks(N: int, chunks: int, align: int = 256, first_weight: float = 1.0):
    """Split [0, N) into <= `chunks` column blocks, each a multiple of `align`
    (the 3xTF32 tile width and the 256-column packB padding unit).  With
    first_weight < 1 the first block is that fraction of the others: it is
    the one whose broadcast nothing overlaps, so it should arrive early."""
    units = (N + align - 1) // align
    chunks = max(1, min(chunks, units))
    w = [first_weight] + [1.0] * (chunks - 1)
    tot = sum(w)
    bounds, acc = [0], 0.0
    for x in w[:-1]:
        acc += x
        b = int(round(units * acc / tot))
        bounds.append(min(max(b, bounds[-1] + 1), units - (chunks - len(bounds))))
    bounds.append(units)
    out = []
    for u0, u1 in zip(bounds[:-1], bounds[1:]):
        n0, n1 = u0 * align, min(u1 * align, N)
        if n1 > n0:
            out.append((n0, n1))
    return out


class PipelinedRowShardGemm:
    """The production multi-GPU step: packedB broadcast in column chunks,
    overlapped with the GEMM on the chunks that already arrived.

    configs[3] ("row-sharded ... with NCCL broadcast of packedB over NVLink"):
      rank src : packB(B[:, chunk c]) -> P_c   (compute stream)
      all      : broadcast(P_c) on NCCL's stream (async, issued in order)
      all      : wait(P_c) -> C[:, chunk c] = A_shard . B[:, chunk c]
                 SIMT (variant 6): elv_gemm_prepacked on the packed chunk
                 3xTF32 / 3xFP16 (variants 7 / 8): split_b_packed(P_c) on a
                 side stream as soon as P_c lands (overlapping the GEMM of
                 chunk c-1), then gemm_planes + the range-guard fix-up
                 (elv_tc_fixup, which reads the fp32 chunk P_c); A's planes
                 are made once per step while chunk 0 is in flight.  Every
                 rank receives fp32 packedB -- the same 4 B per element as
                 fp16 hi/lo planes, half the tf32 planes' -- so every rank
                 can recompute guarded columns.
    The first chunk is half the size of the others (nothing hides its
    broadcast); with 4 chunks and N = 32768 the rest are 37 units of 256
    columns, i.e. 16*37 = 592 = 8 full waves of 74 pair tiles per GEMM at 8
    ranks (4096 rows each).  Column blocks of C are independent, so the
    result is bit-identical to the unchunked kernel's for the same per-tile
    arithmetic.
    """

    def __init__(self, plan, N: int, K: int, device, group=None, src: int = 0, chunks: int = 4,
                 stream=None):
        from . import _lib
        self.lib = _lib.load()
        self._check = _lib.check
        self.plan, self.N, self.K, self.group, self.src = plan, N, K, group, src
        self.variant = plan.variant
        if self.variant not in (4, 5, 6, 7, 8):
            raise ValueError("the pipelined row shard runs the packed / tensor-core variants (4..8)")
        self.device = device
        self.stream = stream or torch.cuda.current_stream(device)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.chunks = column_chunks(N, chunks, first_weight=0.5 if chunks > 1 else 1.0)
        M = plan.M
        if self.variant == 8 and not all(self.lib.elv_fp16x3_applicable(max(M, 1), n1 - n0, K)
                                         for n0, n1 in self.chunks):
            self.variant = 7                        # chunk GEMMs too small for the fp16 encoding
        tc = self.variant in (7, 8)
        # NCCL bytes per step (packB writes whole 256-column groups)
        self.broadcast_bytes = (sum(((n1 - n0 + 255) // 256) * 256 * K * 4 for n0, n1 in self.chunks)
                                if self.world > 1 else 0)
        self.prep = torch.cuda.Stream(device) if tc else None
        self.P = torch.empty(self.lib.elv_pack_b_bytes(K, N) // 4, device=device, dtype=torch.float32)
        if tc:
            pa = self.lib.elv_fp16x3_a_planes_bytes if self.variant == 8 else self.lib.elv_tf32x3_a_planes_bytes
            pb = self.lib.elv_fp16x3_b_planes_bytes if self.variant == 8 else self.lib.elv_tf32x3_b_planes_bytes
            self.a_planes = torch.empty(pa(max(M, 1), K), device=device, dtype=torch.uint8)
            self.b_planes = [torch.empty(pb(n1 - n0, K), device=device, dtype=torch.uint8) for n0, n1 in self.chunks]
        # kernels per step on this rank: pack (src only) + split_a + per chunk
        # (split_b [fp16: column maxima + split] + gemm + fix-up | gemm)
        per_chunk = (4 if self.variant == 8 else 3) if tc else 1
        self.launches = (len(self.chunks) if self.rank == src else 0) + (1 if tc else 0) + \
            per_chunk * len(self.chunks)

    def _panel(self, n0: int) -> torch.Tensor:
        return self.P[(n0 // 32) * self.K * 32:]

    def step(self, A_shard: torch.Tensor, B: torch.Tensor | None, C_shard: torch.Tensor,
             b_ready=None, a_ready=None, chunk_done=None):
        """One step.  Optional hooks for the end-to-end path (host operands):
        b_ready[c] -- event after which B's columns of chunk c are on the
        device (rank src); a_ready -- event for A_shard; chunk_done(c, n0, n1,
        event) is called after chunk c's GEMM is enqueued, with an event
        recorded after it (to start that chunk's D2H)."""
        lib, K, N, st = self.lib, self.K, self.N, self.stream.cuda_stream
        M = A_shard.shape[0]
        works = []
        with torch.cuda.stream(self.stream):
            for c, (n0, n1) in enumerate(self.chunks):
                Pc = self._panel(n0)
                count = ((n1 - n0 + 255) // 256) * 256 * K     # packB writes whole 256-col groups
                if self.rank == self.src and b_ready is not None:
                    self.stream.wait_event(b_ready[c])
                if self.rank == self.src:
                    self._check(lib.elv_pack_b(B.data_ptr() + 4 * n0, Pc.data_ptr(), K, n1 - n0, B.stride(0),
                                               32, st), "elv_pack_b")
                if self.world > 1:
                    works.append(dist.broadcast(Pc[:count], src=self.src, group=self.group, async_op=True))
                else:
                    works.append(None)
            if M == 0:
                for w in works:
                    if w is not None:
                        w.wait()
                return C_shard
            if self.variant in (7, 8):
                f16 = self.variant == 8
                split_b = lib.elv_fp16x3_split_b_packed if f16 else lib.elv_tf32x3_split_b_packed
                split_a = lib.elv_fp16x3_split_a if f16 else lib.elv_tf32x3_split_a
                gemm = lib.elv_fp16x3_gemm_planes if f16 else lib.elv_tf32x3_gemm_planes
                # side stream: split each packed chunk as soon as it lands (after
                # the previous step's GEMMs are done with the plane buffers)
                self.prep.wait_stream(self.stream)
                ready = []
                with torch.cuda.stream(self.prep):
                    pst = self.prep.cuda_stream
                    for (n0, n1), w, bp in zip(self.chunks, works, self.b_planes):
                        if w is not None:
                            w.wait()                # the prep stream waits for chunk c
                        self._check(split_b(self._panel(n0).data_ptr(), K, n1 - n0, bp.data_ptr(), pst),
                                    "split_b_packed")
                        ev = torch.cuda.Event()
                        ev.record(self.prep)
                        ready.append(ev)
                if a_ready is not None:
                    self.stream.wait_event(a_ready)
                ap = self.a_planes.data_ptr()
                self._check(split_a(A_shard.data_ptr(), M, K, A_shard.stride(0), ap, st), "split_a")
                for c, ((n0, n1), bp, ev) in enumerate(zip(self.chunks, self.b_planes, ready)):
                    self.stream.wait_event(ev)
                    Cc = C_shard.data_ptr() + 4 * n0
                    self._check(gemm(ap, bp.data_ptr(), Cc, M, n1 - n0, K, C_shard.stride(0), st), "gemm_planes")
                    self._check(lib.elv_tc_fixup(self.variant, ap, bp.data_ptr(), A_shard.data_ptr(),
                                                 A_shard.stride(0), self._panel(n0).data_ptr(), 0, 1, Cc,
                                                 C_shard.stride(0), M, n1 - n0, K, st), "tc_fixup")
                    self._done(chunk_done, c, n0, n1)
                return C_shard
            if a_ready is not None:
                self.stream.wait_event(a_ready)
            for c, ((n0, n1), w) in enumerate(zip(self.chunks, works)):
                if w is not None:
                    w.wait()                        # compute stream waits for chunk c only
                self._check(lib.elv_gemm_prepacked(self.variant, A_shard.data_ptr(), self._panel(n0).data_ptr(),
                                                   C_shard.data_ptr() + 4 * n0, M, n1 - n0, K, A_shard.stride(0),
                                                   C_shard.stride(0), st), "elv_gemm_prepacked")
                self._done(chunk_done, c, n0, n1)
        return C_shard

    def _done(self, chunk_done, c, n0, n1):
        if chunk_done is not None:
            ev = torch.cuda.Event()
            ev.record(self.stream)
            chunk_done(c, n0, n1, ev)



class HostRowShardPipeline:
    """End to end from host buffers on N GPUs (one process per GPU): rank
    `src` streams B to its device column chunk by column chunk (each chunk is
    packed and NCCL-broadcast as soon as it lands), every rank streams in its
    A shard, and each column chunk of the C shard goes back to the host as
    soon as its GEMM is done -- PCIe in, NVLink and PCIe out overlap the
    GEMMs.  Wraps a PipelinedRowShardGemm; A_dev/B_dev/C_dev are its device
    buffers (B_dev only on `src`)."""

    def __init__(self, pipe: PipelinedRowShardGemm):
        self.pipe = pipe
        self.lib = pipe.lib
        self.s_in = torch.cuda.Stream(pipe.device)
        self.s_out = torch.cuda.Stream(pipe.device)

    def __call__(self, A_h, B_h, C_h, A_dev, B_dev, C_dev, sync: bool = True):
        pipe, lib, st = self.pipe, self.lib, self.pipe.stream
        N, K, rows = pipe.N, pipe.K, A_dev.shape[0]
        for t, shape in ((A_h, (rows, K)), (C_h, (rows, N))):
            if t.is_cuda or tuple(t.shape) != shape or t.stride(-1) != 1 or t.stride(0) != shape[1]:
                raise ValueError(f"host buffers must be contiguous row-major {shape}")
        self.s_in.wait_stream(st)
        self.s_out.wait_stream(st)
        src = pipe.rank == pipe.src
        b_evs = [] if src else None
        a_ev = torch.cuda.Event()
        with torch.cuda.stream(self.s_in):
            for c, (n0, n1) in enumerate(pipe.chunks):
                if src:
                    pipe._check(lib.elv_copy2d(B_dev.data_ptr() + 4 * n0, B_dev.stride(0) * 4,
                                               B_h.data_ptr() + 4 * n0, B_h.stride(0) * 4, (n1 - n0) * 4, K, 1,
                                               self.s_in.cuda_stream), "elv_copy2d")
                    b_evs.append(torch.cuda.Event())
                    b_evs[-1].record(self.s_in)
                if c == 0:
                    # A's event right after its copy: chunk 0's split/GEMM must
                    # not wait for the whole of B to cross PCIe
                    if rows:
                        A_dev.copy_(A_h, non_blocking=True)
                    a_ev.record(self.s_in)

        def chunk_done(c, n0, n1, ev):
            self.s_out.wait_event(ev)
            pipe._check(lib.elv_copy2d(C_h.data_ptr() + 4 * n0, C_h.stride(0) * 4, C_dev.data_ptr() + 4 * n0,
                                       C_dev.stride(0) * 4, (n1 - n0) * 4, rows, 2, self.s_out.cuda_stream),
                        "elv_copy2d")

        pipe.step(A_dev, B_dev, C_dev, b_ready=b_evs, a_ready=a_ev, chunk_done=chunk_done)
        st.wait_stream(self.s_out)
        if sync:
            st.synchronize()
        return C_h


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
