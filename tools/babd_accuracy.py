import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, paper_0912_3678_b200 as psg
for N, p in [(1 << 12, 64), (1 << 14, 64), (1 << 14, 1024), (1 << 16, 256), (1 << 16, 1024), (1 << 18, 256),
             (1 << 18, 1024), (1 << 18, 4096)]:
    A, f = psg.generate_config(4, N, 5)
    F = psg.parallel_factor(A, p)
    x = psg.solve(F, f)
    res = psg.residual(A, x, f)
    Ah = O.Matrix(A.kind, A.n, A.m, A.s, A.r, A.data.cpu().numpy(), A.corner.cpu().numpy(), 8, 8)
    xs = O.solve_sequential(Ah, f.cpu().numpy())
    line = f"N={N:7d} p={p:5d} gpu residual {res:.2e}  rel diff vs seq {O.rel_err(x.cpu().numpy(), xs):.2e}"
    if N <= 1 << 14 and p <= 1024:
        xp, _ = O.parallel_solve(Ah, p, f.cpu().numpy())
        line += f"  | ref-par residual {O.residual(Ah, xp, f.cpu().numpy()):.2e}"
    print(line, flush=True)
