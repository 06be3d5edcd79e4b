"""Host<->device copy bandwidth on the box: H2D, D2H, and both at once.

Sizes the e2e pipeline (interp.HostPipeline): pinned host buffers, CUDA
events on the copy streams."""
import json

import torch


def main():
    dev = torch.device("cuda", 0)
    n = 1 << 28  # 1 GiB of fp32
    h_in = torch.empty(n, pin_memory=True)
    h_out = torch.empty(n, pin_memory=True)
    d_in = torch.empty(n, device=dev)
    d_out = torch.empty(n, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}

    def timed(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    def h2d():
        s1.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    def d2h_chunked(chunks=16):
        s2.wait_stream(torch.cuda.current_stream())
        c = n // chunks
        with torch.cuda.stream(s2):
            for i in range(chunks):
                h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)

    for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("d2h_16chunks", d2h_chunked)):
        ms = timed(fn)
        gb = (2 if name == "both" else 1) * 4 * n / 1e9
        res[name] = {"ms": round(ms, 3), "GB/s": round(gb / (ms / 1e3), 2)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
