"""Parareal (§8(f) row 4) measurement: psg_parareal_solve (libparsol_b200 ->
psg_pr_*: fine propagations one warp per window, coarse sweep on the device)
against the unmodified reference parareal_solve (oracle/_ref, OpenMP over the
host threads) on the 1-D heat problem (reference heat_problem), optionally
forced by the compiled C callback of tools/ode_forcing.c.

  python tools/pr_bench.py [--m 64 --p 64 --N 1000 --coarse-steps 1 --reps 3]"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=64)
    ap.add_argument("--p", type=int, default=64)
    ap.add_argument("--N", type=int, default=1000)
    ap.add_argument("--T", type=float, default=0.1)
    ap.add_argument("--coarse-steps", type=int, default=1)
    ap.add_argument("--method", type=int, default=0)
    ap.add_argument("--forced", action="store_true")
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    import oracle as O
    from ode_bench import forcing_lib
    m, p, N = a.m, a.p, a.N
    inv = float(m + 1) ** 2
    L = np.ascontiguousarray(np.diag(-2.0 * inv * np.ones(m)) + np.diag(inv * np.ones(m - 1), 1) +
                             np.diag(inv * np.ones(m - 1), -1))
    y0 = np.sin(np.pi * np.arange(1, m + 1) / (m + 1))
    g = C.cast(forcing_lib().ode_forcing, C.c_void_p) if a.forced else None
    mctx = C.c_int(m)
    cfg = {"workload": "Parareal, 1-D heat problem", "m": m, "p": p, "N": N, "T": a.T,
           "fine": ["ie", "trap"][a.method] + f"x{N}", "coarse": f"ie x{a.coarse_steps}", "forced": a.forced,
           "tol": a.tol}

    def run(lib, fn):
        inits = np.zeros(p * m)
        hist = np.zeros(4 * p)
        it, conv = C.c_int(), C.c_int()
        err = C.create_string_buffer(256)
        rc = getattr(lib, fn)(C.c_int(m), L.ctypes.data_as(C.c_void_p), y0.ctypes.data_as(C.c_void_p),
                              C.c_double(0.0), C.c_double(a.T), C.c_int(p), C.c_int(N), g,
                              C.byref(mctx) if g else None, C.c_int(0), C.c_int(a.method), C.c_int(N), C.c_int(1),
                              C.c_int(0), C.c_int(a.coarse_steps), C.c_double(a.tol), C.c_int(-1),
                              inits.ctypes.data_as(C.c_void_p), hist.ctypes.data_as(C.c_void_p), C.c_int(4 * p),
                              C.byref(it), C.byref(conv), err, C.c_size_t(256))
        assert rc == 0, err.value
        return inits, it.value, conv.value

    def timed(fn, reps):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = fn()
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts)), r

    ours = C.CDLL(os.path.join(ROOT, "paper_0912_3678_b200", "libparsol_b200.so"))
    t, (x, it, conv) = timed(lambda: run(ours, "psg_parareal_solve"), a.reps)
    print(json.dumps({"impl": "ours", "metric": "fine_steps_per_s", "value": (p - 1) * N * it / t, "ms": t * 1e3,
                      "iterations": it, "converged": conv, "config": cfg}))
    if a.no_ref:
        return
    ref = O.ref()
    t, (xr, itr, convr) = timed(lambda: run(ref, "ref_parareal_solve"), 1)
    print(json.dumps({"impl": "reference", "metric": "fine_steps_per_s", "value": (p - 1) * N * itr / t,
                      "ms": t * 1e3, "iterations": itr, "converged": convr, "cores": os.cpu_count(),
                      "rel_diff_vs_ours": O.rel_err(x, xr), "config": cfg}))


if __name__ == "__main__":
    main()
