"""Small driver for ncu captures: one config instance, W factor+solve steps."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0912_3678_b200 as psg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--size", type=int, default=1 << 26)
ap.add_argument("--p", type=int, default=65536)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
A, f = psg.generate_config(a.config, a.size, 2)
x = torch.empty_like(f)
for _ in range(a.steps):
    F = psg.parallel_factor(A, a.p)
    st = psg.SolveStats()
    psg.solve(F, f, st, x=x)
    F.close()
torch.cuda.synchronize()
print("ok", st.as_dict())
