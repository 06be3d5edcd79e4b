"""GPU: GEMMs on concurrent streams.  The tcgen05 kernels pace their TMA
producers with a wave counter in device memory, zeroed on the launch stream;
each (device, stream) has its own counter, so a launch on one stream never
zeroes the counter under a multi-wave kernel running on another."""

import pytest
import torch

from paper_2002_02268_b200 import interp, schedules, synth

pytestmark = pytest.mark.gpu


def _call(shape, enc, seed, stream, dev):
    M, N, K = shape
    p = interp.plan(schedules.apply_padded("parallel", M, N, K).term, [(M, K), (K, N)], True, enc)
    A = torch.empty((M, K), device=dev); synth.fill_device(A, seed, 0)
    B = torch.empty((K, N), device=dev); synth.fill_device(B, seed, 1)
    C = torch.empty((M, N), device=dev)
    return interp.GemmCall(p, A, B, C, stream)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("enc", ["fp16", "tf32"])
def test_multiwave_gemms_on_concurrent_streams(cuda, enc):
    """A long multi-wave pair-kernel GEMM and short multi-wave GEMMs launched
    on other streams while it runs: every result equals its serial run."""
    s_big, s_a, s_b = (torch.cuda.Stream(cuda) for _ in range(3))
    big = _call((8192, 8192, 2048), enc, 21, s_big, cuda)           # 1024 pair tiles, ~14 waves
    small = [_call((2560, 2816, 1024), enc, 22 + i, s, cuda) for i, s in enumerate((s_a, s_b))]
    torch.cuda.synchronize()                    # inputs were filled on the default stream
    ref = []
    for c in [big, *small]:
        c()
        torch.cuda.synchronize()
        ref.append(c.C.clone())
    for _ in range(3):
        for c in [big, *small]:
            c.C.fill_(float("nan"))
        torch.cuda.synchronize()
        big()                                   # enqueued first, runs while the small ones start
        for _ in range(4):
            for c in small:
                c()
        torch.cuda.synchronize()
        for c, r in zip([big, *small], ref):
            assert torch.equal(c.C, r)
