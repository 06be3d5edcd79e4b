"""CPU, world_size 2 over gloo: the row-shard driver's host logic.

The GEMM itself is injected (f64 oracle) because there is no GPU here; the
product path computes with the CUDA kernels (see paper_2002_02268_b200/
distributed.py).  What is tested: the shard partition, the broadcast of B
from rank 0, and that the assembled C equals the unsharded result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2002_02268_b200 import distributed as D
from paper_2002_02268_b200 import synth


@pytest.mark.parametrize("M,world", [(32768, 8), (32768, 2), (1000, 3), (100, 4), (1, 2), (129, 2)])
def test_shard_rows_partition(M, world):
    shards = [D.shard_rows(M, world, r) for r in range(world)]
    assert shards[0].row0 == 0
    for a, b in zip(shards, shards[1:]):
        assert a.row0 + a.rows == b.row0
    assert sum(s.rows for s in shards) == M
    for s in shards[:-1]:
        if s.rows and shards[-1].rows:
            assert s.rows % D.ROW_ALIGN == 0
    if M % (world * D.ROW_ALIGN) == 0:
        assert all(s.rows == M // world for s in shards)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, M, N, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = D.shard_rows(M, world, rank, align=8)
        A_shard = torch.from_numpy(synth.matrix(sh.rows, K, 0, 0, row0=sh.row0))
        # B only exists on rank 0; the others receive it
        B = torch.from_numpy(synth.matrix(K, N, 0, 1)) if rank == 0 else torch.zeros((K, N))
        C_shard = torch.empty((sh.rows, N), dtype=torch.float32)

        def cpu_compute(A, B, C):       # injected: the test's stand-in for the kernel
            C.copy_(torch.from_numpy((A.double().numpy() @ B.double().numpy()).astype(np.float32)))
            return C

        g = D.RowShardGemm(compute=cpu_compute)
        g.step(A_shard, B, C_shard)
        full = D.gather_rows(C_shard, M, align=8)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,N,K", [(40, 24, 16), (17, 8, 8)])
def test_rowshard_gloo_world2(M, N, K):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, N, K, q)) for r in range(2)]
    for p in procs:
        p.start()
    C = q.get(timeout=90)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = synth.matrix(M, K, 0, 0).astype(np.float64)
    B = synth.matrix(K, N, 0, 1).astype(np.float64)
    assert np.array_equal(C, (A @ B).astype(np.float32))


@pytest.mark.parametrize("N,chunks", [(32768, 4), (2048, 4), (1000, 3), (256, 8), (300, 4), (4096, 1)])
def test_column_chunks_partition(N, chunks):
    """Broadcast chunks: a partition of [0, N) into 256-aligned blocks (but the
    tail), at most `chunks` of them, the first about half the others."""
    cs = D.column_chunks(N, chunks, first_weight=0.5)
    assert cs[0][0] == 0 and cs[-1][1] == N and len(cs) <= chunks
    assert all(a[1] == b[0] for a, b in zip(cs, cs[1:]))
    assert all(n0 % 256 == 0 and n1 > n0 for n0, n1 in cs)
    if N == 32768 and chunks == 4:
        assert [(n1 - n0) // 256 for n0, n1 in cs] == [18, 37, 36, 37]
