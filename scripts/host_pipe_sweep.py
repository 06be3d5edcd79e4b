"""e2e host pipeline (elv_gemm_host) tile-shape sweep at the bench shape, plus
2D-copy bandwidth of one C tile.  Timing: wall clock around synchronised
calls (the e2e definition), best of 3 after one warm-up."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402


def main():
    M, N, K = 32768, 32768, 8192
    dev = torch.device("cuda", 0)
    tf = "--simt" not in sys.argv
    term = schedules.apply("parallel", M, N, K).term
    p = dispatch.decode(term, [(M, K), (K, N)], tf32x3=tf)
    A_d = torch.empty((M, K), device=dev)
    B_d = torch.empty((K, N), device=dev)
    synth.fill_device(A_d, 0, 0)
    synth.fill_device(B_d, 0, 1)
    A = torch.empty((M, K), pin_memory=True)
    B = torch.empty((K, N), pin_memory=True)
    A.copy_(A_d)
    B.copy_(B_d)
    del A_d, B_d
    C = torch.empty((M, N), pin_memory=True)

    # 2D D2H / H2D of one 4096 x 8192 tile out of a 32768-wide matrix vs contiguous
    lib = interp._lib.load()
    Cd = torch.empty((4096, N), device=dev)
    res = {}
    for name, fn in (
        ("d2h_tile_2d_4096x8192", lambda: C[:4096, :8192].copy_(Cd[:, :8192], non_blocking=True)),
        ("d2h_rows_4096x8192_contig", lambda: C.view(-1)[:4096 * 8192].copy_(Cd.view(-1)[:4096 * 8192], non_blocking=True)),
    ):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        res[name] = {"ms": dt * 1e3, "GB/s": 4 * 4096 * 8192 / dt / 1e9}
    del Cd
    print(json.dumps(res), flush=True)

    tiles = os.environ.get("SWEEP_TILES", "None,4096:4096,2048:8192,8192:4096,2048:4096,4096:16384,8192:8192").split(",")
    tiles = [None if t == "None" else t.replace(":", ",") for t in tiles]
    nds = os.environ.get("SWEEP_D2H", "").split(",") if os.environ.get("SWEEP_D2H") else [None]
    for nd, t in [(nd, t) for nd in nds for t in tiles]:
        if nd:
            os.environ["ELV_HOST_D2H_STREAMS"] = nd
        if t:
            os.environ["ELV_HOST_TILES"] = t
        else:
            os.environ.pop("ELV_HOST_TILES", None)
        interp._host_pipes.clear()
        torch.cuda.empty_cache()
        hp = interp.HostPipeline(p, dev)
        hp(A, B, C)
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            hp(A, B, C)
            best = min(best, time.perf_counter() - t0)
        print(json.dumps({"tiles": hp.tile, "d2h_streams": nd, "ms": best * 1e3,
                          "TFLOP/s": 2.0 * M * N * K / best / 1e12}), flush=True)
        del hp


if __name__ == "__main__":
    main()
