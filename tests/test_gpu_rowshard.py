"""GPU: the pipelined row-shard driver (chunked packedB broadcast + GEMM).

Only one GPU exists here, so (a) the chunked pipeline is checked at world 1
(no collective) against the unchunked kernel -- bit-identical, since column
blocks of C do the same per-tile arithmetic -- and (b) two ranks share cuda:0
over gloo (which broadcasts CUDA tensors) to exercise the async broadcast /
per-chunk wait logic across processes.  NCCL itself needs one GPU per rank.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

from paper_2002_02268_b200 import dispatch, distributed as D, interp, schedules, synth

pytestmark = pytest.mark.gpu


def _plan(variant, M, N, K):
    sched, tf = ("parallel", True) if variant == 7 else ("parallel", False)
    p = dispatch.decode(schedules.apply_padded(sched, M, N, K).term, [(M, K), (K, N)], tf32x3=tf)
    return p


@pytest.mark.parametrize("variant", [6, 7])
@pytest.mark.parametrize("shape,chunks", [((512, 2048, 512), 4), ((300, 1000, 200), 3), ((128, 256, 64), 8)])
def test_pipelined_world1_bitwise_equals_direct(cuda, variant, shape, chunks):
    M, N, K = shape
    p = _plan(variant, M, N, K)
    A = torch.empty((M, K), device=cuda); synth.fill_device(A, 3, 0)
    B = torch.empty((K, N), device=cuda); synth.fill_device(B, 3, 1)
    C_direct = interp.gemm(p, A, B)
    pipe = D.PipelinedRowShardGemm(p, N, K, cuda, chunks=chunks)
    C = torch.full((M, N), float("nan"), device=cuda)
    pipe.step(A, B, C)
    torch.cuda.synchronize()
    assert torch.equal(C, C_direct)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, variant, M, N, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        sh = D.shard_rows(M, world, rank)
        p = _plan(variant, M, N, K)
        import dataclasses
        p = dataclasses.replace(p, M=sh.rows)
        A = torch.empty((max(sh.rows, 1), K), device=dev)[:sh.rows]
        if sh.rows:
            synth.fill_device(A, 0, 0, offset=sh.row0 * K)
        B = None
        if rank == 0:
            B = torch.empty((K, N), device=dev)
            synth.fill_device(B, 0, 1)
        C = torch.zeros((sh.rows, N), device=dev)
        pipe = D.PipelinedRowShardGemm(p, N, K, dev, chunks=3)
        pipe.step(A, B, C)
        torch.cuda.synchronize()
        q.put((rank, sh.row0, C.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", [6, 7])
def test_two_ranks_share_one_gpu_over_gloo(cuda, variant):
    M, N, K = 384, 1024, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, variant, M, N, K, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    parts = sorted([q.get(timeout=240) for _ in range(2)])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    C = np.concatenate([c for _, _, c in parts], 0)
    # the same rows from one unsharded launch
    p = _plan(variant, M, N, K)
    A = torch.empty((M, K), device=cuda); synth.fill_device(A, 0, 0)
    B = torch.empty((K, N), device=cuda); synth.fill_device(B, 0, 1)
    ref = interp.gemm(p, A, B).cpu().numpy()
    assert np.array_equal(C, ref)


@pytest.mark.parametrize("tiles", [None, "384,1280"])
@pytest.mark.parametrize("variant", ["baseline", "loopPerm", "arrayPacking", "parallel", "parallel_tf32x3"])
def test_host_pipeline_bitwise_equals_device_path(cuda, variant, tiles, monkeypatch):
    """interp.run on host tensors through the C-ABI host pipeline
    (elv_gemm_host: tiles of C with overlapped H2D / GEMM / D2H) returns
    exactly the single-launch result -- with the default tiling and with a
    forced 384 x 1280 tiling that leaves ragged row and column tails."""
    sched, tf = ("parallel", True) if variant == "parallel_tf32x3" else (variant, False)
    M, N, K = 1100, 4096, 2048
    if variant == "baseline":
        M, N, K = 1100, 4096, 512
    from paper_2002_02268_b200 import interp as I
    monkeypatch.setattr(I, "_PIPELINE_MIN_BYTES", 1 << 20)
    if tiles:
        monkeypatch.setenv("ELV_HOST_TILES", tiles)
    I._host_pipes.clear()
    term = schedules.apply_padded(sched, M, N, K).term
    A = torch.from_numpy(synth.matrix(M, K, 8, 0)).pin_memory()
    B = torch.from_numpy(synth.matrix(K, N, 8, 1)).pin_memory()
    C_host = I.run(term, [A, B], tf32x3=tf)
    assert not C_host.is_cuda
    p = I.plan(term, [(M, K), (K, N)], tf)         # the same plan (default encoding) run() used
    if tiles:
        assert I._host_pipes and next(iter(I._host_pipes.values())).tile == (384, 1280)
    C_dev = I.gemm(p, A.to(cuda), B.to(cuda)).cpu()
    assert torch.equal(C_host, C_dev)
    I._host_pipes.clear()


def test_host_pipeline_large_default_tiling(cuda, monkeypatch):
    """The default tiling at a bench-like shape (8 row blocks; N < 32768, so
    one column chunk) and repeated calls reusing the cached workspace: row samples
    against the f64 oracle, and call 2 == call 1."""
    from paper_2002_02268_b200 import interp as I
    M, N, K = 4096, 16384, 1024
    monkeypatch.setenv("ELV_HOST_PLAN", "grid")     # N >= 16384 would take the growing schedule
    I._host_pipes.clear()
    term = schedules.apply("parallel", M, N, K).term
    A = torch.from_numpy(synth.matrix(M, K, 9, 0)).pin_memory()
    B = torch.from_numpy(synth.matrix(K, N, 9, 1)).pin_memory()
    C1 = torch.empty((M, N), pin_memory=True)
    I.run(term, [A, B], tf32x3=True, out=C1)
    (hp,) = [h for k, h in I._host_pipes.items() if k[1:4] == (M, N, K)]
    assert hp.tile == (512, 16384)
    C2 = torch.empty((M, N), pin_memory=True)
    I.run(term, [A, B], tf32x3=True, out=C2)
    assert torch.equal(C1, C2)
    rows = np.r_[0:4, 511:514, M - 3:M]
    An, Bn = A.numpy(), B.numpy()
    ok, worst = oracle.check(C1.numpy()[rows], oracle.mm_f64(An[rows], Bn), oracle.absprod_np(An[rows], Bn), K)
    assert ok, worst
    I._host_pipes.clear()


def test_c_abi_rowshard_single_process(cuda):
    """elv_gemm_rowshard (one process, ncclCommInitAll) over the devices we
    have (1 here): NCCL broadcast of B + pack + GEMM on each shard."""
    import ctypes
    from paper_2002_02268_b200 import _lib
    lib = _lib.load()
    ndev = 1
    devs = (ctypes.c_int * ndev)(*range(ndev))
    _lib.check(lib.elv_nccl_init(ndev, devs), "elv_nccl_init")
    try:
        M, N, K = 384, 640, 200
        A = torch.empty((M, K), device=cuda); synth.fill_device(A, 6, 0)
        B = torch.empty((K, N), device=cuda); synth.fill_device(B, 6, 1)
        P = torch.empty(lib.elv_pack_b_bytes(K, N) // 4, device=cuda)
        C = torch.empty((M, N), device=cuda)
        vp = ctypes.c_void_p
        arr = lambda *xs: (vp * ndev)(*xs)
        rows = (ctypes.c_int * ndev)(M)
        stream = torch.cuda.current_stream().cuda_stream
        rc = lib.elv_gemm_rowshard(6, ndev, devs, arr(A.data_ptr()), arr(B.data_ptr()), arr(P.data_ptr()),
                                   arr(C.data_ptr()), rows, N, K, arr(stream))
        _lib.check(rc, "elv_gemm_rowshard")
        torch.cuda.synchronize()
        ref = interp.gemm(_plan(6, M, N, K), A, B)
        assert torch.equal(C, ref)
    finally:
        lib.elv_nccl_destroy()


@pytest.mark.parametrize("ranks,shape", [(2, ("2048", "2048", "1024")), (4, ("4096", "32768", "1024"))],
                         ids=["2ranks", "4ranks-fp16"])
def test_bench_ranks_sharing_one_gpu(cuda, tmp_path, ranks, shape):
    """bench.py's N>1 path (torchrun, PipelinedRowShardGemm, barriers,
    max-over-ranks timing, rank-0 JSON line) with 2 and 4 ranks sharing cuda:0
    over gloo (ELV_BENCH_SHARE_GPU=1, test-only); NCCL itself needs one GPU
    per rank."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ELV_BENCH_SHARE_GPU="1")
    M, N, K = shape
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(repo, "bench.py"),
           "--gpus", str(ranks), "--M", M, "--N", N, "--K", K, "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=repo)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == ranks and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == f"rowshard{ranks}"


def test_host_pipeline_concurrent_callers(cuda):
    """Two Python threads on two streams sharing one cached host pipeline
    (same plan -> same workspace): calls are serialised on the workspace, and
    both results are exact."""
    import threading
    from paper_2002_02268_b200 import interp as I
    M, N, K = 1024, 2048, 512
    term = schedules.apply("parallel", M, N, K).term
    ins = [(torch.from_numpy(synth.matrix(M, K, s, 0)).pin_memory(),
            torch.from_numpy(synth.matrix(K, N, s, 1)).pin_memory()) for s in (21, 22)]
    p = dispatch.decode(term, [(M, K), (K, N)], tf32x3=True)
    refs = [I.gemm(p, A.to(cuda), B.to(cuda)).cpu() for A, B in ins]
    hp = I.host_pipeline(p, cuda)
    outs = [torch.empty((M, N), pin_memory=True) for _ in ins]
    errs = []

    def work(i):
        try:
            s = torch.cuda.Stream(cuda)
            with torch.cuda.stream(s):
                for _ in range(3):
                    hp(ins[i][0], ins[i][1], outs[i])
        except Exception as e:      # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    for o, r in zip(outs, refs):
        assert torch.equal(o, r)


def _worker_host(rank, world, port, variant, M, N, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        sh = D.shard_rows(M, world, rank)
        import dataclasses
        p = dataclasses.replace(_plan(variant, M, N, K), M=sh.rows)
        A_h = torch.from_numpy(synth.matrix(sh.rows, K, 5, 0, row0=sh.row0)).pin_memory()
        B_h = torch.from_numpy(synth.matrix(K, N, 5, 1)).pin_memory() if rank == 0 else None
        C_h = torch.full((sh.rows, N), float("nan")).pin_memory()
        A = torch.empty((sh.rows, K), device=dev)
        B = torch.empty((K, N), device=dev) if rank == 0 else None
        C = torch.empty((sh.rows, N), device=dev)
        pipe = D.PipelinedRowShardGemm(p, N, K, dev, chunks=3)
        hp = D.HostRowShardPipeline(pipe)
        for _ in range(2):                              # reuse of every buffer
            hp(A_h, B_h, C_h, A, B, C)
        q.put((rank, sh.row0, C_h.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", [6, 7])
def test_host_row_shard_pipeline_two_ranks(cuda, variant):
    """The multi-GPU end-to-end path from host buffers (B streamed to rank 0 by
    column chunk and broadcast chunk by chunk, C chunks streamed back) with
    two ranks sharing cuda:0 over gloo: the gathered C equals one unsharded
    launch bit for bit."""
    M, N, K = 384, 1280, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_host, args=(r, 2, port, variant, M, N, K, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    parts = sorted([q.get(timeout=240) for _ in range(2)])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    C = np.concatenate([c for _, _, c in parts], 0)
    p = _plan(variant, M, N, K)
    A = torch.from_numpy(synth.matrix(M, K, 5, 0)).to(cuda)
    B = torch.from_numpy(synth.matrix(K, N, 5, 1)).to(cuda)
    assert np.array_equal(C, interp.gemm(p, A, B).cpu().numpy())


def _plan16(M, N, K):
    return dispatch.decode(schedules.apply_padded("parallel", M, N, K).term, [(M, K), (K, N)], tf32x3=True,
                           tc_encoding="fp16")


def test_fp16x3_pipelined_and_host_paths_bitwise(cuda, monkeypatch):
    """The 3xFP16 encoding through the chunked row-shard pipeline (planes
    prepared per column chunk on the source rank) and through the host
    pipeline (planes per tile) equals the single launch bit for bit: the
    per-row / per-column scales do not depend on the tiling."""
    from paper_2002_02268_b200 import interp as I
    M, N, K = 8192, 16384, 1024
    p = _plan16(M, N, K)
    assert p.variant == 8
    A = torch.empty((M, K), device=cuda); synth.fill_device(A, 9, 0)
    B = torch.empty((K, N), device=cuda); synth.fill_device(B, 9, 1)
    direct = I.gemm(p, A, B)
    pipe = D.PipelinedRowShardGemm(p, N, K, cuda, chunks=4)
    assert pipe.variant == 8
    C = torch.full((M, N), float("nan"), device=cuda)
    pipe.step(A, B, C)
    torch.cuda.synchronize()
    assert torch.equal(C, direct)
    monkeypatch.setenv("ELV_HOST_TILES", "2048,8192")
    I._host_pipes.clear()
    hp = I.HostPipeline(p, cuda)
    assert hp.tile == (2048, 8192)
    out = torch.empty((M, N), pin_memory=True)
    hp(A.cpu().pin_memory(), B.cpu().pin_memory(), out)
    assert torch.equal(out, direct.cpu())
    I._host_pipes.clear()


@pytest.mark.parametrize("enc", ["tf32", "fp16"])
@pytest.mark.parametrize("strips", [None, "384,1280", "256,8192"])
def test_host_pipeline_growing_schedule_bitwise(cuda, enc, strips, monkeypatch):
    """The growing schedule (strips of A and B prepared into full-size plane
    buffers, each landed strip multiplied against the other operand's resident
    prefix) returns exactly the single-launch result: default strips, ragged
    strips, and strips wider than the matrix."""
    from paper_2002_02268_b200 import interp as I
    M, N, K = 3000, 5000, 640
    p = dispatch.decode(schedules.apply_padded("parallel", M, N, K).term, [(M, K), (K, N)], tf32x3=True,
                        tc_encoding=enc)
    monkeypatch.setenv("ELV_HOST_PLAN", "grow")
    if strips:
        monkeypatch.setenv("ELV_HOST_STRIPS", strips)
    I._host_pipes.clear()
    hp = I.HostPipeline(p, cuda)
    if strips:
        r, c = map(int, strips.split(","))
        assert hp.tile == (min(r, M), min(c, N))
    A = torch.empty((M, K), device=cuda); synth.fill_device(A, 11, 0)
    B = torch.empty((K, N), device=cuda); synth.fill_device(B, 11, 1)
    direct = I.gemm(p, A, B).cpu()
    out = torch.full((M, N), float("nan")).pin_memory()
    for _ in range(2):                      # the second call reuses the workspace
        hp(A.cpu().pin_memory(), B.cpu().pin_memory(), out)
        assert torch.equal(out, direct)
    I._host_pipes.clear()


def test_host_pipeline_grows_at_bench_scale(cuda):
    """Large outputs take the growing schedule by default (1024-row and
    4096-column strips) and match the f64 oracle on sampled rows."""
    from paper_2002_02268_b200 import interp as I
    M, N, K = 16384, 16384, 1024
    p = _plan16(M, N, K)
    I._host_pipes.clear()
    hp = I.HostPipeline(p, cuda)
    assert hp.tile == (1024, 4096)
    A = torch.empty((M, K), device=cuda); synth.fill_device(A, 12, 0)
    B = torch.empty((K, N), device=cuda); synth.fill_device(B, 12, 1)
    out = torch.empty((M, N), pin_memory=True)
    hp(A.cpu().pin_memory(), B.cpu().pin_memory(), out)
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    rows = np.array([0, 1023, 1024, 8191, 16383])
    ref = oracle.mm_f64(Ah[rows], Bh)
    ok, worst = oracle.check(out.numpy()[rows], ref, oracle.absprod_np(Ah[rows], Bh), K)
    assert ok, worst
    assert torch.equal(out, I.gemm(p, A, B).cpu())
    I._host_pipes.clear()


def test_bench_gpus_flag_launches_ranks_itself(cuda):
    """`python bench.py --gpus 2` with no launcher around it re-runs itself
    under torch.distributed.run (one rank per GPU; here the two ranks share
    cuda:0 over gloo, ELV_BENCH_SHARE_GPU=1) and rank 0 prints the one JSON
    line: n_gpus 2, per-rank step times (max over ranks = ms_per_step) and
    the broadcast bytes per step."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["ELV_BENCH_SHARE_GPU"] = "1"
    cmd = [sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--M", "2048", "--N", "4096",
           "--K", "1024", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=repo)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "rowshard2"
    assert d["ranks"]["world_size"] == 2 and len(d["ranks"]["per_rank_ms_per_step"]) == 2
    assert abs(max(d["ranks"]["per_rank_ms_per_step"]) - d["ms_per_step"]) < 1e-6
    assert d["ranks"]["broadcast_bytes_per_step"] == 4096 * 1024 * 4
    assert "with 2 ranks" in r.stderr


def _rowshard_pipelined(lib, variant, devs, A_list, B_root, rows, N, K, chunks, streams):
    """Call elv_gemm_rowshard_pipelined over len(devs) devices; returns the C shards."""
    import ctypes
    from paper_2002_02268_b200 import _lib
    nd = len(devs)
    vp = ctypes.c_void_p
    cdevs = (ctypes.c_int * nd)(*devs)
    P = [torch.empty(lib.elv_pack_b_bytes(K, N) // 4, device=torch.device("cuda", d)) for d in devs]
    C = [torch.empty((r, N), device=torch.device("cuda", d)) for r, d in zip(rows, devs)]
    wsb = lib.elv_gemm_rowshard_workspace_bytes(variant, max(rows), N, K, chunks)
    W = [torch.empty(max(wsb, 1), dtype=torch.uint8, device=torch.device("cuda", d)) for d in devs]
    arr = lambda xs: (vp * nd)(*[x.data_ptr() for x in xs])  # noqa: E731
    rc = lib.elv_gemm_rowshard_pipelined(variant, nd, cdevs, arr(A_list), B_root.data_ptr(), arr(P), arr(C),
                                         (ctypes.c_int * nd)(*rows), N, K, chunks, arr(W), wsb,
                                         (vp * nd)(*streams))
    _lib.check(rc, "elv_gemm_rowshard_pipelined")
    for d in devs:
        torch.cuda.synchronize(d)
    return C


@pytest.mark.parametrize("variant", [6, 7, 8])
@pytest.mark.parametrize("chunks", [1, 4])
def test_c_abi_pipelined_rowshard_bitwise(cuda, variant, chunks):
    """elv_gemm_rowshard_pipelined (one process, ncclCommInitAll, chunked
    packedB broadcast, split-on-arrival, GEMM + range-guard fix-up per chunk)
    at ndev = 1: bitwise elv_gemm of the same variant, also with a guarded
    row (the fix-up reads the broadcast packedB chunk)."""
    import ctypes
    from paper_2002_02268_b200 import _lib
    lib = _lib.load()
    devs = [0]
    _lib.check(lib.elv_nccl_init(1, (ctypes.c_int * 1)(0)), "elv_nccl_init")
    try:
        M, N, K = 768, 2304, 1024
        A = torch.empty((M, K), device=cuda); synth.fill_device(A, 8, 0)
        B = torch.empty((K, N), device=cuda); synth.fill_device(B, 8, 1)
        A[17, 5] = 2.0 ** -110                        # a range-guarded row for 7 / 8
        st = torch.cuda.current_stream().cuda_stream
        (C,) = _rowshard_pipelined(lib, variant, devs, [A], B, [M], N, K, chunks, [st])
        ref = interp.gemm(_plan16(M, N, K) if variant == 8 else _plan(variant, M, N, K), A, B)
        torch.cuda.synchronize()
        assert torch.equal(C, ref)
    finally:
        lib.elv_nccl_destroy()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("variant", [6, 7, 8])
def test_c_abi_pipelined_rowshard_two_devices(cuda, variant):
    """Two devices in one process: each shard bitwise equal to elv_gemm on it."""
    import ctypes
    from paper_2002_02268_b200 import _lib
    lib = _lib.load()
    devs = [0, 1]
    _lib.check(lib.elv_nccl_init(2, (ctypes.c_int * 2)(*devs)), "elv_nccl_init")
    try:
        M, N, K = 1024, 4096, 1024
        rows = [512, 512]
        A = torch.empty((M, K), device=cuda); synth.fill_device(A, 9, 0)
        B = torch.empty((K, N), device=cuda); synth.fill_device(B, 9, 1)
        A_list = [A[:512].contiguous(), A[512:].to("cuda:1")]
        streams = [torch.cuda.current_stream(0).cuda_stream, torch.cuda.current_stream(1).cuda_stream]
        C0, C1 = _rowshard_pipelined(lib, variant, devs, A_list, B, rows, N, K, 4, streams)
        ref = interp.gemm(_plan16(M, N, K) if variant == 8 else _plan(variant, M, N, K), A, B)
        torch.cuda.synchronize()
        assert torch.equal(C0, ref[:512]) and torch.equal(C1.cpu(), ref[512:].cpu())
    finally:
        lib.elv_nccl_destroy()
