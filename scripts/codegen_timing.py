"""Generated-kernel (codegen.py) timing vs the template kernels, for DESIGN:
the general compiler is the correct-by-construction path for schedules the
templates do not know; this measures what that generality costs."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02268_b200 import codegen, interp, schedules, synth  # noqa: E402


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = int(os.environ.get("N", 1024))
    dev = torch.device("cuda", 0)
    A = torch.empty((n, n), device=dev); B = torch.empty((n, n), device=dev)
    synth.fill_device(A, 0, 0); synth.fill_device(B, 0, 1)
    from paper_2002_02268_b200._ref import S
    st, nf, tv, rules = S().strategy, S().normal_forms, S().traversals, S().rules
    # a user schedule outside the seven templates: tile(16,16) + split(2) of the reduce, no reorder
    user = st.seq(nf.dfnf_seq(tv.top_down(schedules.tile(16, 16)),
                              tv.top_down(st.seq(tv.is_reduce, rules.make_split(2)))), nf.LOWER_TO_C)
    terms = [("user_tile16_split2", st.run_strategy(user, schedules.mm(n, n, n))[0].term)]
    user2 = st.seq(nf.dfnf_seq(tv.top_down(schedules.tile(32, 64)),
                               tv.top_down(st.seq(tv.is_reduce, rules.make_split(8)))), nf.LOWER_TO_C)
    terms += [("user_tile32x64_split8", st.run_strategy(user2, schedules.mm(n, n, n))[0].term)]
    terms += [(name, schedules.apply(name, n, n, n).term) for name in schedules.SCHEDULE_NAMES]
    for name, term in terms:
        t0 = time.perf_counter()
        codegen.run(term, [A, B]); torch.cuda.synchronize()
        compile_s = time.perf_counter() - t0
        g = timed(lambda: codegen.run(term, [A, B]))
        mode = codegen.kernel_for(term).c.mode
        if name.startswith("user"):
            t, diff = None, None
            ref = A.double() @ B.double()
            diff = (codegen.run(term, [A, B]).double() - ref).abs().max().item()
        else:
            t = timed(lambda: interp.run_tensor(term, A, B))
            diff = (codegen.run(term, [A, B]) - interp.run_tensor(term, A, B)).abs().max().item()
        print(json.dumps({"schedule": name, "n": n, "mode": mode, "generated_ms": g, "template_ms": t,
                          "generated_gflops": 2 * n ** 3 / g / 1e6,
                          "template_gflops": 2 * n ** 3 / t / 1e6 if t else None,
                          "first_call_s": compile_s, "max_abs_diff": diff}), flush=True)


if __name__ == "__main__":
    main()
