"""Cycle accounting of the 1-CTA tensor-core kernel (k7_tf32x3<BN, BK, F16>,
small problems) in the -DELV_K7_PROF tuning build: where the producer, MMA
issuer and epilogue threads spend their cycles at 1024^3 (tuning evidence).

    python scripts/k7_prof_small.py --build    # here (no GPU)
    python scripts/k7_prof_small.py            # on the GPU box
"""
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
    n = int(os.environ.get("N", 1024))
    M = N = K = n
    lib = _lib.load()
    lib.elv_debug_k7_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
    dev = torch.device("cuda", 0)
    A = torch.empty((M, K), device=dev); B = torch.empty((K, N), device=dev)
    synth.fill_device(A, 0, 0); synth.fill_device(B, 0, 1)
    C = torch.empty((M, N), device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for enc in ("fp16", "tf32"):
        pre = "elv_fp16x3_" if enc == "fp16" else "elv_tf32x3_"
        ap = torch.empty(getattr(lib, pre + "a_planes_bytes")(M, K), dtype=torch.uint8, device=dev)
        bp = torch.empty(getattr(lib, pre + "b_planes_bytes")(N, K), dtype=torch.uint8, device=dev)
        _lib.check(getattr(lib, pre + "split_a")(A.data_ptr(), M, K, K, ap.data_ptr(), st), "a")
        _lib.check(getattr(lib, pre + "split_b")(B.data_ptr(), K, N, N, bp.data_ptr(), st), "b")
        host = np.zeros((512, 12), np.uint64)
        for rep in range(4):
            lib.elv_debug_k7_prof(host.ctypes.data, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(getattr(lib, pre + "gemm_planes")(ap.data_ptr(), bp.data_ptr(), C.data_ptr(), M, N, K, N, st),
                       "g")
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            lib.elv_debug_k7_prof(host.ctypes.data, 0)
            h = host.astype(np.float64)
            used = h[h[:, 7] > 0]                      # CTAs that ran tiles (MMA thread counted them)
            tot = used[:, 2].mean()
            clk = float(torch.cuda.clock_rate()) if hasattr(torch.cuda, "clock_rate") else None
            out = {"enc": enc, "n": n, "us": 1e3 * ms, "TF": 2.0 * M * N * K / ms / 1e9, "ctas": int(len(used)),
                   "mma_loop_cyc": tot, "prologue_cyc": used[:, 11].mean(),
                   "mma_wait_tempty_frac": used[:, 0].mean() / tot, "mma_wait_full_frac": used[:, 1].mean() / tot,
                   "prod_wait_empty_frac": used[:, 3].mean() / tot,
                   "epi_wait_tfull_frac": used[:, 5].mean() / tot, "epi_store_cyc": used[:, 6].mean(),
                   "chunks_per_cta": used[:, 9].mean(), "sm_clock_khz": clk}
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
