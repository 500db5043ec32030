"""Config-1 step-time decomposition: full step vs parts (timing experiment)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0912_3678_b200 as psg  # noqa: E402

A, f = psg.generate_config(1, 1 << 26, 2)
x = torch.empty_like(f)
H = psg.parallel_factor(A, 65536)


def run(label, fn, steps=20):
    for _ in range(3):
        fn()
    H.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    H.sync()
    e1.record()
    torch.cuda.synchronize()
    print("%-40s %8.1f us/step" % (label, e0.elapsed_time(e1) / steps * 1e3), flush=True)


run("refactor + solve_async(timing)", lambda: (H.refactor(A), H.solve_async(f, x, timing=True)))
run("refactor + solve_async", lambda: (H.refactor(A), H.solve_async(f, x)))
run("solve_async only", lambda: H.solve_async(f, x))
run("refactor only", lambda: H.refactor(A))
