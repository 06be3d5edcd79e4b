"""Rewrite-step table for the seven GEMM schedules (
PAPER.md:359-368 Fig. rewrite-steps), with the reference's ExecContext counters.

    python -m paper_2002_02268_b200.steps [M N K]
"""

from __future__ import annotations

import sys
import time

from . import schedules
from ._ref import S

PAPER_STEPS = {"baseline": 211, "blocking": 92980, "vectorized": 94030, "loopPerm": 80710,
               "arrayPacking": 143270, "cacheBlocks": 144183, "parallel": 144074}


def table(M: int = 1024, N: int = 1024, K: int = 1024):
    s = S()
    rows = []
    for name in schedules.SCHEDULE_NAMES:
        t0 = time.perf_counter()
        res, ctx = s.strategy.run_strategy(schedules.strategy(name), schedules.mm(M, N, K))
        dt = time.perf_counter() - t0
        rows.append({"schedule": name, "ok": isinstance(res, s.strategy.Success),
                     "rule_successes": ctx.total, "committed": ctx.committed_count,
                     "per_rule": dict(ctx.per_rule), "seconds": round(dt, 3),
                     "paper_scala_elevate": PAPER_STEPS[name]})
    return rows


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    M, N, K = (int(x) for x in argv[:3]) if len(argv) >= 3 else (1024, 1024, 1024)
    print(f"{'schedule':14s} {'successes':>9s} {'seconds':>8s} {'paper (Scala ELEVATE)':>22s}")
    for r in table(M, N, K):
        print(f"{r['schedule']:14s} {r['rule_successes']:9d} {r['seconds']:8.3f} {r['paper_scala_elevate']:22d}")


if __name__ == "__main__":
    main()
