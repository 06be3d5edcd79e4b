"""Cycle accounting of k7_tf32x3_pair (tuning build with -DELV_K7_PROF).

Builds the instrumented library next to the product one, runs the bench-shape
GEMM (3xTF32 planes) and prints where the MMA issuer, producer and epilogue
threads spend their cycles."""
import ctypes
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
PROF_LIB = os.path.join(REPO, "paper_2002_02268_b200", "libelevate_b200_prof.so")
if "--build" in sys.argv:
    from paper_2002_02268_b200 import build
    build.build(force=True, defines=("ELV_K7_PROF",), out=PROF_LIB, verbose=False)
    sys.exit(0)
os.environ["ELV_LIB"] = PROF_LIB

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_02268_b200 import _lib, synth  # noqa: E402


def main():
    M = N = int(os.environ.get("N", 32768)); K = int(os.environ.get("K", 8192))
    lib = _lib.load()
    lib.elv_debug_k7_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
    dev = torch.device("cuda", 0)
    A = torch.empty((M, K), device=dev); B = torch.empty((K, N), device=dev)
    synth.fill_device(A, 0, 0); synth.fill_device(B, 0, 1)
    f16 = os.environ.get("ENC", "fp16") == "fp16"
    pre = "elv_fp16x3_" if f16 else "elv_tf32x3_"
    ap = torch.empty(getattr(lib, pre + "a_planes_bytes")(M, K), dtype=torch.uint8, device=dev)
    bp = torch.empty(getattr(lib, pre + "b_planes_bytes")(N, K), dtype=torch.uint8, device=dev)
    C = torch.empty((M, N), device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(getattr(lib, pre + "split_a")(A.data_ptr(), M, K, K, ap.data_ptr(), st), "a")
    _lib.check(getattr(lib, pre + "split_b")(B.data_ptr(), K, N, N, bp.data_ptr(), st), "b")
    host = np.zeros((512, 12), np.uint64)
    for rep in range(3):
        lib.elv_debug_k7_prof(host.ctypes.data, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(getattr(lib, pre + "gemm_planes")(ap.data_ptr(), bp.data_ptr(), C.data_ptr(), M, N, K, N, st), "g")
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        lib.elv_debug_k7_prof(host.ctypes.data, 0)
        h = host.astype(np.float64)
        lead = h[0:296:2]; both = h[:296]
        tot = lead[:, 2].mean()
        out = {"ms": ms, "TF": 2.0 * M * N * K / ms / 1e9,
               "mma_total_cyc": tot,
               "mma_wait_tempty_frac": lead[:, 0].mean() / tot,
               "mma_wait_full_frac": lead[:, 1].mean() / tot,
               "tiles_per_cluster": lead[:, 7].mean(),
               "prod_wait_empty_frac": both[:, 3].mean() / tot,
               "prod_wave_sync_frac": both[:, 4].mean() / tot,
               "epi_wait_tfull_frac": both[:, 5].mean() / tot,
               "epi_store_frac": both[:, 6].mean() / tot,
               "epi_store_cyc_per_tile": both[:, 6].mean() / max(1, lead[:, 7].mean()),
               "epi_chunk_drain_cyc": both[:, 8].sum() / max(1, both[:, 9].sum()),
               "epi_chunk_wait_cyc": both[:, 5].sum() / max(1, both[:, 9].sum()),
               "epi_chunk_arrive_cyc": both[:, 10].sum() / max(1, both[:, 9].sum()),
               "mma_cyc_per_chunk": tot / max(1, lead[:, 7].mean() * K / (64 if f16 else 32)),
               "mma_wait_full_max_frac": (lead[:, 1] / lead[:, 2]).max()}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
