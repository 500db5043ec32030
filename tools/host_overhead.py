"""Per-step host overhead: factor+solve on a tiny system (device work ~ few us)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0912_3678_b200 as psg  # noqa: E402

A, f = psg.generate_config(1, 1 << 16, 2)
x = torch.empty_like(f)
for _ in range(20):
    F = psg.parallel_factor(A, 64)
    psg.solve(F, f, psg.SolveStats(), x=x)
    F.close()
torch.cuda.synchronize()
for label, stats in (("with stats", True), ("no stats", False)):
    t0 = time.perf_counter()
    N = 200
    for _ in range(N):
        F = psg.parallel_factor(A, 64)
        psg.solve(F, f, psg.SolveStats() if stats else None, x=x)
        F.close()
    dt = (time.perf_counter() - t0) / N
    print(f"{label}: {dt * 1e6:.1f} us per factor+solve (n=2^16, p=64)")
t0 = time.perf_counter()
for _ in range(200):
    F = psg.parallel_factor(A, 64)
    F.close()
torch.cuda.synchronize()
print(f"factor only: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")

# production loop (bench.py other_configs): refactor + async solve per step,
# host time to enqueue vs. device time per step, config-0 size
A0, f0 = psg.generate_config(0, 1 << 20, 1)
x0 = torch.empty_like(f0)
H = psg.parallel_factor(A0, 1024)
for _ in range(20):
    H.refactor(A0)
    H.solve_async(f0, x0)
H.sync()
torch.cuda.synchronize()
for timing in (False, True):
    N = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(N):
        H.refactor(A0)
        H.solve_async(f0, x0, timing=timing)
    t1 = time.perf_counter()
    H.sync()
    e1.record()
    torch.cuda.synchronize()
    print(f"cfg0 refactor+solve_async (timing={timing}): host enqueue {(t1 - t0) / N * 1e6:.1f} us/step, "
          f"device {e0.elapsed_time(e1) / N * 1e3:.1f} us/step")
