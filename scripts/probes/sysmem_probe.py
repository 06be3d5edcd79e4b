"""PCIe probe for a zero-copy epilogue: SM stores into pinned host memory vs
copy-engine D2H, alone and while a 1 GiB H2D runs on another stream."""
import ctypes
import json
import os

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsysmem_probe.so"))
lib.probe_fill_host.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda", 0)
GB = 1 << 30
host_out = torch.empty(GB // 4, dtype=torch.float32, pin_memory=True)
host_in = torch.empty(GB // 4, dtype=torch.float32, pin_memory=True)
dev_buf = torch.empty(GB // 4, dtype=torch.float32, device=dev)
dev_in = torch.empty(GB // 4, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, concurrent_h2d=False, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        if concurrent_h2d:
            s2.wait_event(e0)
            with torch.cuda.stream(s2):
                dev_in.copy_(host_in, non_blocking=True)
        fn()
        e1.record(s1)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return GB / (best * 1e-3) / 1e9


def sm_store(blocks):
    def f():
        rc = lib.probe_fill_host(host_out.data_ptr(), GB, blocks, s1.cuda_stream)
        assert rc == 0, rc
    return f


def ce_d2h():
    with torch.cuda.stream(s1):
        host_out.copy_(dev_buf, non_blocking=True)


for blocks in (148, 296, 592, 1184):
    print(json.dumps({"path": "sm_store", "blocks": blocks, "GB/s": round(timed(sm_store(blocks)), 1)}))
print(json.dumps({"path": "ce_d2h", "GB/s": round(timed(ce_d2h), 1)}))
for blocks in (296, 1184):
    print(json.dumps({"path": "sm_store+h2d", "blocks": blocks, "GB/s": round(timed(sm_store(blocks), True), 1)}))
print(json.dumps({"path": "ce_d2h+h2d", "GB/s": round(timed(ce_d2h, True), 1)}))
assert float(host_out[12345]) in (0.0, 1.0)
