"""PCIe throughput of 2D (strided) copies vs row width, each direction alone
and with the other direction busy: sizes the host pipeline's tiles (narrow
first chunks start the D2H stream sooner but copy shorter rows).

    python scripts/pcie_2d_probe.py > gpurun_out/pcie_2d.jsonl
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import _lib


def main():
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    pitch = 32768 * 4                     # a 32768-column fp32 matrix
    rows = 8192
    h = torch.empty(rows * 32768, pin_memory=True)
    d = torch.empty(rows * 32768, device=dev)
    h2 = torch.empty(1 << 28, pin_memory=True)
    d2 = torch.empty(1 << 28, device=dev)
    s, s_other = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    for w_cols in (1024, 2048, 4096, 8192, 16384, 32768):
        height = min(rows, (256 << 20) // (w_cols * 4))      # ~256 MB per copy
        for kind, name in ((1, "h2d"), (2, "d2h")):
            for busy in (False, True):
                best = 1e9
                for _ in range(3):
                    torch.cuda.synchronize()
                    if busy:   # the other direction streams 1 GiB meanwhile
                        with torch.cuda.stream(s_other):
                            if kind == 1:
                                h2.copy_(d2, non_blocking=True)
                            else:
                                d2.copy_(h2, non_blocking=True)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    dst, src = (d, h) if kind == 1 else (h, d)
                    rc = lib.elv_copy2d(ctypes.c_void_p(dst.data_ptr()), pitch, ctypes.c_void_p(src.data_ptr()),
                                        pitch, w_cols * 4, height, kind, ctypes.c_void_p(s.cuda_stream))
                    assert rc == 0
                    e1.record(s)
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                gb = w_cols * 4 * height / 1e9
                print(json.dumps({"dir": name, "row_bytes": w_cols * 4, "rows": height, "other_busy": busy,
                                  "ms": round(best, 3), "GB/s": round(gb / (best / 1e3), 2)}), flush=True)


if __name__ == "__main__":
    main()
