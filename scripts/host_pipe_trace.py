"""Timeline of one elv_gemm_host call at the bench shape (ELV_HOST_TRACE=1):
when each H2D item landed, each tile's GEMM finished and each tile's D2H
finished; D2H-stream idle time = where the e2e pipeline loses to PCIe."""
import ctypes
import json
import os
import sys

os.environ["ELV_HOST_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import _lib, dispatch, interp, schedules, synth  # noqa: E402


def main():
    M, N, K = 32768, 32768, 8192
    tf = "--simt" not in sys.argv
    dev = torch.device("cuda", 0)
    p = dispatch.decode(schedules.apply("parallel", M, N, K).term, [(M, K), (K, N)], tf32x3=tf,
                        tc_encoding=os.environ.get("ENC", "fp16"))
    A = torch.empty((M, K), pin_memory=True); B = torch.empty((K, N), pin_memory=True)
    Ad = torch.empty((M, K), device=dev); synth.fill_device(Ad, 0, 0); A.copy_(Ad); del Ad
    Bd = torch.empty((K, N), device=dev); synth.fill_device(Bd, 0, 1); B.copy_(Bd); del Bd
    C = torch.empty((M, N), pin_memory=True)
    hp = interp.HostPipeline(p, dev)
    for _ in range(2):
        hp(A, B, C)
    buf = np.zeros(4096, np.float32)
    n = _lib.load().elv_gemm_host_trace(buf.ctypes.data, 2048)
    ev = buf[:2 * n].reshape(n, 2)
    kinds = {0: "h2d", 1: "gemm", 2: "d2h"}
    out = {k: [round(float(t), 2) for kk, t in ev if int(kk) == i] for i, k in kinds.items()}
    d2h = out["d2h"]
    print(json.dumps({"tiles": hp.tile, "h2d_done_ms": out["h2d"], "gemm_done_ms": out["gemm"],
                      "d2h_done_ms": d2h, "total_ms": d2h[-1] if d2h else None,
                      "first_d2h_ms": d2h[0] if d2h else None}))


if __name__ == "__main__":
    main()
