"""3xFP16 prepare (variant 8) at small/mid shapes under the prepare modes:
ELV_FP16X3_WARP_ROWS (2: warp per A row, row in registers; 1: warp per row,
two passes; 0: block per row) x ELV_FP16X3_COLMAX_SLAB (0: adaptive, 64: the
round-1 fixed slab).  CUDA events, L2 flushed before every rep (as the
ladder), median of 30; prints one JSON line per (shape, mode).

    python scripts/fp16_prep_timing.py
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import interp, schedules, synth  # noqa: E402

MODES = [("1", "64"), ("1", "0"), ("2", "64"), ("2", "0")]


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for M, N, K in ((1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096), (1536, 1536, 1536),
                    (8192, 8192, 8192)):
        A = torch.empty((M, K), device=dev); synth.fill_device(A, 0, 0)
        B = torch.empty((K, N), device=dev); synth.fill_device(B, 0, 1)
        p = interp.plan(schedules.apply_padded("parallel", M, N, K).term, [(M, K), (K, N)], True, "fp16")
        outs = {}
        for wr, slab in MODES:
            os.environ["ELV_FP16X3_WARP_ROWS"], os.environ["ELV_FP16X3_COLMAX_SLAB"] = wr, slab
            call = interp.GemmCall(p, A, B, torch.empty((M, N), device=dev))
            for _ in range(5):
                call()
            prep, tot = [], []
            for _ in range(30):
                flush.zero_()
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record(); call.prepare(); e1.record(); call.compute(); e2.record()
                torch.cuda.synchronize()
                prep.append(e0.elapsed_time(e1) * 1e3); tot.append(e0.elapsed_time(e2) * 1e3)
            outs[(wr, slab)] = call.C.clone()
            us = statistics.median(tot)
            print(json.dumps({"shape": [M, N, K], "warp_rows": int(wr), "colmax_slab": int(slab) or "adaptive",
                              "prepare_us": round(statistics.median(prep), 2), "call_us": round(us, 2),
                              "TFLOP/s_call": round(2.0 * M * N * K / (us * 1e-6) / 1e12, 1)}), flush=True)
        ref = outs[MODES[0]]
        print(json.dumps({"shape": [M, N, K], "bitwise_equal_all_modes": all(torch.equal(ref, o) for o in outs.values())}),
              flush=True)
        os.environ.pop("ELV_FP16X3_WARP_ROWS"); os.environ.pop("ELV_FP16X3_COLMAX_SLAB")


if __name__ == "__main__":
    main()
