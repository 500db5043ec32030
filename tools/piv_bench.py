"""Pivoting strategies (§8(f) row 3) measurement: LuPivot / Qr factor + solve
on the GPU (csrc/piv_kernels.cuh) against the unmodified reference
parallel_factor / solve (oracle/_ref, OpenMP over the host threads), same
matrix, same p, same tol.

  python tools/piv_bench.py [--kind 4 --n 1048576 --s 1 --r 1 --p 1024 --strategy 4 --dom 1.0]

Prints one JSON line per arm (GPU: median over reps; kernel time by CUDA
events around factor+solve with the device-resident matrix and rhs)."""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", type=int, default=4)
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--m", type=int, default=1)
    ap.add_argument("--s", type=int, default=1)
    ap.add_argument("--r", type=int, default=1)
    ap.add_argument("--p", type=int, default=1024)
    ap.add_argument("--strategy", type=int, default=4)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--dom", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ref-n", type=int, default=0, help="reference on a smaller n (0: same n)")
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    import torch
    import oracle as O
    import paper_0912_3678_b200 as psg
    from test_pivot_gpu import ref_random

    A = ref_random(a.kind, a.n, a.m, a.s, a.r, 1234, a.dom)
    f = O.random_vector(a.n, 7)
    dev = lambda v: None if v is None else torch.from_numpy(np.ascontiguousarray(v)).cuda()
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, dev(A.data), dev(A.corner), A.corner_rows, A.corner_cols)
    df = dev(f)
    dx = torch.empty_like(df)
    cfg = {"workload": "pivoting partition solve", "kind": a.kind, "n": a.n, "m": a.m, "s": a.s, "r": a.r,
           "p": a.p, "strategy": {4: "lupivot", 5: "qr"}.get(a.strategy, a.strategy), "tol": a.tol,
           "dominance": a.dom}

    def step():
        F = psg.parallel_factor(GA, a.p, a.strategy, a.tol)
        st = psg.SolveStats()
        psg.solve(F, df, st, x=dx)
        return F, st

    F, st = step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts, tk = [], []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev0.record()
        F, st = step()
        ev1.record()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        tk.append(ev0.elapsed_time(ev1) * 1e-3)
    x = dx.cpu().numpy()
    extras = F.q - (a.p + 1 if F.has_corner else a.p - 1)
    print(json.dumps({"impl": "ours", "metric": "unknowns_per_s", "value": a.n / float(np.median(ts)),
                      "ms": float(np.median(ts)) * 1e3, "ms_events": float(np.median(tk)) * 1e3,
                      "factor_ms": st.factor_seconds * 1e3,
                      "solve_phases_ms": [st.phase1_seconds * 1e3, st.phase2_seconds * 1e3, st.phase3_seconds * 1e3],
                      "reduced_dim": F.dim, "extras": extras, "certificate": st.certificate, "config": cfg}))
    if a.no_ref:
        return
    nref = a.ref_n or a.n
    if nref != a.n:
        A = ref_random(a.kind, nref, a.m, a.s, a.r, 1234, a.dom)
        f = O.random_vector(nref, 7)
    t0 = time.perf_counter()
    R = O.RefMatrix(A).factor_tol(a.p, a.strategy, a.tol)
    t1 = time.perf_counter()
    xr, _, ph = R.solve(f)
    t2 = time.perf_counter()
    out = {"impl": "reference", "metric": "unknowns_per_s", "value": nref / (t2 - t0), "ms": (t2 - t0) * 1e3,
           "factor_ms": (t1 - t0) * 1e3, "solve_ms": (t2 - t1) * 1e3, "cores": os.cpu_count(),
           "sample_n": nref, "config": cfg}
    if nref == a.n:
        out["rel_diff_vs_ours"] = O.rel_err(x, xr)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
