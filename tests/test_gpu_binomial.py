"""GPU: binomial-filter kernels through the C ABI against the oracle."""

import json
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2002_02268_b200 import binomial, interp, synth

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(GOLD, "golden.json")))["bf_cases"]


def _check(out, ref, img):
    err = np.abs(np.asarray(out, np.float64) - ref)
    b = oracle.bf_bound(img)
    assert np.all(err <= b), f"worst err/bound {float((err / np.maximum(b, 1e-300)).max()):.3g}"


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_bf_golden(cuda, case):
    z = np.load(os.path.join(GOLD, case["name"] + ".npz"))
    img = z["img"]
    for name in binomial.SCHEDULE_NAMES:
        t = binomial.apply(name, case["H"], case["W"])
        out = interp.run(t, [img])                       # numpy in, numpy out
        _check(out, z[name], img)
    # lists in -> lists out, like the reference
    t = binomial.apply("separatedPar", case["H"], case["W"])
    lst = interp.run(t, [img.tolist()])
    assert isinstance(lst, list) and len(lst) == case["H"]


@pytest.mark.parametrize("shape", [(1, 1), (1, 300), (300, 1), (33, 257), (257, 513), (1000, 1000),
                                   (4096, 4096)], ids=lambda s: f"{s[0]}x{s[1]}")
def test_bf_sizes_and_band_equivalence(cuda, shape):
    H, W = shape
    img = torch.empty((H, W), device=cuda)
    synth.fill_device(img, 4, 2)
    outs = {}
    for name in binomial.SCHEDULE_NAMES:
        out = torch.empty_like(img)
        binomial.launch(binomial.VARIANTS[name], img, out)
        outs[name] = out
    h = img.cpu().numpy()
    _check(outs["naive"].cpu().numpy(), oracle.bf_interp_f64(h, "naive"), h)
    _check(outs["separated"].cpu().numpy(), oracle.bf_interp_f64(h, "separated"), h)
    # the banded (mapPar) kernels do the same per-pixel arithmetic
    assert torch.equal(outs["naivePar"], outs["naive"])
    assert torch.equal(outs["separatedPar"], outs["separated"])


def test_bf_strided_input(cuda):
    big = torch.empty((50, 80), device=cuda)
    synth.fill_device(big, 2, 2)
    img = big[3:43, 5:70]
    out = torch.full((40, 66), -1.0, device=cuda)[:, :65]
    binomial.launch(binomial.VARIANTS["separatedPar"], img, out)
    h = img.cpu().numpy()
    _check(out.cpu().numpy(), oracle.bf_interp_f64(h, "separated"), h)
