"""e2e host pipeline (elv_gemm_host) at the bench shape: the grid plan vs
the growing schedule with several strip sizes.  Wall clock around
synchronised calls (the e2e definition), best of 3 after one warm-up.

    ENC=fp16 python scripts/host_plan_sweep.py > gpurun_out/host_plan_sweep.jsonl
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import dispatch, interp, schedules, synth  # noqa: E402


def main():
    M, N, K = (int(x) for x in os.environ.get("SHAPE", "32768,32768,8192").split(","))
    enc = os.environ.get("ENC", "fp16")
    dev = torch.device("cuda", 0)
    p = dispatch.decode(schedules.apply_padded("parallel", M, N, K).term, [(M, K), (K, N)], tf32x3=True,
                        tc_encoding=enc)
    A_d = torch.empty((M, K), device=dev); synth.fill_device(A_d, 0, 0)
    B_d = torch.empty((K, N), device=dev); synth.fill_device(B_d, 0, 1)
    A = torch.empty((M, K), pin_memory=True); A.copy_(A_d)
    B = torch.empty((K, N), pin_memory=True); B.copy_(B_d)
    del A_d, B_d
    C = torch.empty((M, N), pin_memory=True)
    configs = os.environ.get("CONFIGS", "grid:-,grow:-,grow:512:2048,grow:2048:2048,grow:1024:4096,grow:1024:1024")
    for cfg in configs.split(","):
        plan, *strip = cfg.split(":")
        os.environ["ELV_HOST_PLAN"] = plan
        if len(strip) == 3:                 # grow:R:Nc:rows-per-D2H-copy
            os.environ["ELV_HOST_D2H_ROWS"] = strip.pop()
        else:
            os.environ.pop("ELV_HOST_D2H_ROWS", None)
        if strip and strip[0] != "-":
            os.environ["ELV_HOST_STRIPS"] = ",".join(strip)
        else:
            os.environ.pop("ELV_HOST_STRIPS", None)
        interp._host_pipes.clear()
        torch.cuda.empty_cache()
        hp = interp.HostPipeline(p, dev)
        hp(A, B, C)
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            hp(A, B, C)
            best = min(best, time.perf_counter() - t0)
        print(json.dumps({"shape": [M, N, K], "enc": enc, "plan": plan, "tiles": hp.tile,
                          "d2h_rows": os.environ.get("ELV_HOST_D2H_ROWS"), "pace": os.environ.get("ELV_HOST_PACE"), "ms": round(best * 1e3, 2),
                          "TFLOP/s": round(2.0 * M * N * K / best / 1e12, 1)}), flush=True)
        del hp


if __name__ == "__main__":
    main()
