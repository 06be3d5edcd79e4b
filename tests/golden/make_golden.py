"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference or baseline/_ref):

    python tests/golden/make_golden.py

For every case it applies the schedule with the reference's own rules, runs
the reference interpreter `stratir.interp.run` (reference
pkg/src/stratir/interp.py:157-162) on seeded synthetic inputs
(paper_2002_02268_b200.synth, exact in fp32 and f64) and stores inputs,
output (f64, exactly what the interpreter returned), the schedule name, the
shapes and the rule-success count.  The fixtures pin both the C oracle
(bit-exact) and the GPU kernels (within the fp32 bound) without needing the
reference at test time.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
if os.path.isdir("/root/reference/pkg/src"):
    sys.path.insert(0, "/root/reference/pkg/src")   # the reference, read-only

from paper_2002_02268_b200 import schedules, synth  # noqa: E402
from paper_2002_02268_b200._ref import S  # noqa: E402

# (case name, schedule, true M, N, K) -- terms are built at the padded shape
CASES = [(f"{s}_64x96x64", s, 64, 96, 64) for s in schedules.SCHEDULE_NAMES]
CASES += [
    ("baseline_5x7x3", "baseline", 5, 7, 3),
    ("blocking_pad_40x36x22", "blocking", 40, 36, 22),
    ("parallel_pad_33x40x20", "parallel", 33, 40, 20),
    ("arrayPacking_pad_31x65x33", "arrayPacking", 31, 65, 33),
]


def run_case(name, sched, M, N, K, seed=7):
    s = S()
    sc = schedules.apply_padded(sched, M, N, K)
    Mp, Np, Kp = sc.M, sc.N, sc.K
    A = synth.matrix(M, K, seed, 0)
    B = synth.matrix(K, N, seed, 1)
    Ap = np.zeros((Mp, Kp), np.float32); Ap[:M, :K] = A
    Bp = np.zeros((Kp, Np), np.float32); Bp[:K, :N] = B
    t0 = time.time()
    C = np.array(s.interp.run(sc.term, [Ap.tolist(), Bp.tolist()]), np.float64)[:M, :N]
    dt = time.time() - t0
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), A=A, B=B, C=C)
    return {"name": name, "schedule": sched, "M": M, "N": N, "K": K,
            "term_shape": [Mp, Np, Kp], "seed": seed,
            "rule_successes": sc.rule_successes, "interp_seconds": round(dt, 2),
            "macs": Mp * Np * Kp}


BF_CASES = [(1, 1), (2, 3), (7, 9), (24, 40)]


def run_bf_cases():
    """Binomial-filter schedules through the reference interpreter."""
    from paper_2002_02268_b200 import binomial
    s = S()
    out = []
    for H, W in BF_CASES:
        img = synth.matrix(H, W, 9, 2)
        res = {}
        for name in binomial.SCHEDULE_NAMES:
            t = binomial.apply(name, H, W)
            res[name] = np.array(s.interp.run(t, [img.tolist()]), np.float64)
        fname = f"bf_{H}x{W}"
        np.savez_compressed(os.path.join(HERE, f"{fname}.npz"), img=img, **res)
        out.append({"name": fname, "H": H, "W": W, "seed": 9})
    return out


def kats():
    """Known answers from the reference SPEC, evaluated by the interpreter."""
    s = S()
    out = {}
    t = schedules.apply("baseline", 1, 1, 3).term
    out["dot_1x3x1"] = s.interp.run(t, [[[1.0, 2.0, 3.0]], [[4.0], [5.0], [6.0]]])  # SPEC.md:214 -> 32
    t = schedules.apply("baseline", 2, 3, 2).term
    B = [[1.5, -2.0, 0.25], [3.0, 0.5, -1.0]]
    out["identity_2x3x2"] = {"B": B, "C": s.interp.run(t, [[[1.0, 0.0], [0.0, 1.0]], B])}
    return out


def main():
    meta = {"cases": [], "kats": kats(), "bf_cases": run_bf_cases()}
    for c in CASES:
        info = run_case(*c)
        print(info, flush=True)
        meta["cases"].append(info)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
