"""Time-parallel IVP measurement (§8(f) row 2): psg_ode_solve (libparsol_b200:
host window discretisation + psg_ode_trajectory on the GPU) against the
unmodified reference solve_ivp_parallel / solve_ivp_sequential (oracle/_ref,
OpenMP over all host threads), same problem, same C forcing callback.

  python tools/ode_bench.py [--m 8 --p 4096 --N 64 --method 1 --reps 5]

Prints one JSON line per arm plus the max relative difference between them."""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def forcing_lib():
    out = os.path.join(ROOT, "tools", "_build", "libode_forcing.so")
    src = os.path.join(ROOT, "tools", "ode_forcing.c")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", out, src, "-lm"], check=True)
    return C.CDLL(out)


def step_backward_error(traj, L, y0, T, p, N, m, method):
    """max over all p N steps of the componentwise backward error of
    diag y_k = sub y_{k-1} + rhs_k (numpy restatement of the forcing)."""
    h = T / (p * N)  # uniform windows of equal length: every h_i equals this up to rounding
    I = np.eye(m)
    D, S = (I - h * L, I) if method == 0 else (I - h / 2 * L, I + h / 2 * L)
    Y = traj.reshape(p * N + 1, m)
    t = np.arange(1, p * N + 1) * h
    q = np.arange(1, m + 1)
    g = lambda tt: np.sin(np.outer(tt, q)) + 0.5 * np.cos(2.0 * tt)[:, None]
    rhs = h * g(t) if method == 0 else h / 2 * (g(t - h) + g(t))
    r = Y[1:] @ D.T - Y[:-1] @ S.T - rhs
    den = np.abs(Y[1:]) @ np.abs(D).T + np.abs(Y[:-1]) @ np.abs(S).T + np.abs(rhs)
    return float(np.max(np.abs(r) / den))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--p", type=int, default=4096)
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--method", type=int, default=1)
    ap.add_argument("--T", type=float, default=4.0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    m, p, N = a.m, a.p, a.N
    rng = np.random.default_rng(5)
    L = np.ascontiguousarray(rng.uniform(-1, 1, (m, m)) - 2.0 * np.eye(m))
    y0 = rng.uniform(-1, 1, m)
    fl = forcing_lib()
    gptr = C.cast(fl.ode_forcing, C.c_void_p)
    mctx = C.c_int(m)
    out = np.zeros((p * N + 1) * m)
    err = C.create_string_buffer(256)
    ours = C.CDLL(os.path.join(ROOT, "paper_0912_3678_b200", "libparsol_b200.so"))
    cert = C.c_double()

    def run_ours():
        rc = ours.psg_ode_solve(C.c_int(m), L.ctypes.data_as(C.c_void_p), y0.ctypes.data_as(C.c_void_p),
                                C.c_double(0.0), C.c_double(a.T), C.c_int(p), C.c_int(N), C.c_int(a.method), gptr,
                                C.byref(mctx), out.ctypes.data_as(C.c_void_p), C.byref(cert), err, C.c_size_t(256))
        assert rc == 0, err.value

    def timed(fn):
        fn()
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts))

    cfg = {"workload": "linear IVP y'=Ly+g(t)", "m": m, "p": p, "N": N, "steps": p * N,
           "method": ["ie", "trap"][a.method], "T": a.T}
    t = timed(run_ours)
    mine = out.copy()
    print(json.dumps({"impl": "ours", "metric": "ivp_steps_per_s", "value": p * N / t, "ms": t * 1e3,
                      "certificate": cert.value,
                      "step_backward_error": step_backward_error(mine, L, y0, a.T, p, N, m, a.method), "config": cfg, "path": "psg_ode_solve (host discretise + GPU)"}))
    # the device part alone: psg_ode_trajectory from prepared window blocks
    h = a.T / (p * N)
    I = np.eye(m)
    D, S = (I - h * L, I) if a.method == 0 else (I - h / 2 * L, I + h / 2 * L)
    win = np.ascontiguousarray(np.broadcast_to(np.stack([D, S]), (p, 2, m, m)))
    g = np.concatenate([y0, rng.uniform(-1, 1, p * N * m)])
    psg = C.CDLL(os.path.join(ROOT, "paper_0912_3678_b200", "libpsg.so"))

    class Stats(C.Structure):
        _fields_ = [("factor_seconds", C.c_double), ("p1", C.c_double), ("p2", C.c_double), ("p3", C.c_double),
                    ("ops", C.c_longlong), ("certificate", C.c_double), ("spec", C.c_int), ("fallbacks", C.c_int)]
    st = Stats()
    traj = np.zeros_like(out)

    def run_traj():
        rc = psg.psg_ode_trajectory(C.c_int(m), C.c_int(p), C.c_int(N), win.ctypes.data_as(C.c_void_p),
                                    g.ctypes.data_as(C.c_void_p), traj.ctypes.data_as(C.c_void_p), None,
                                    C.byref(st), err, C.c_size_t(256))
        assert rc == 0, err.value
    t = timed(run_traj)
    print(json.dumps({"impl": "ours", "path": "psg_ode_trajectory (upload + GPU + download)", "ms": t * 1e3,
                      "h2d_bytes": win.nbytes + g.nbytes, "d2h_bytes": traj.nbytes,
                      "gpu_factor_solve_ms": (st.factor_seconds + st.p1 + st.p2 + st.p3) * 1e3, "config": cfg}))
    if a.no_ref:
        return
    import oracle as O
    ref = O.ref()
    ncores = os.cpu_count()
    ref_par = None
    for parallel in (1, 0):
        def run_ref():
            rc = ref.ref_ode_solve(C.c_int(m), L.ctypes.data_as(C.c_void_p), y0.ctypes.data_as(C.c_void_p),
                                   C.c_double(0.0), C.c_double(a.T), C.c_int(p), C.c_int(N), C.c_int(a.method), gptr,
                                   C.byref(mctx), C.c_int(parallel), out.ctypes.data_as(C.c_void_p), err,
                                   C.c_size_t(256))
            assert rc == 0, err.value
        t = timed(run_ref)
        d = float(np.max(np.abs(out - mine)) / np.max(np.abs(out)))
        extra = {}
        if ref_par is None:
            ref_par = out.copy()
        else:  # the reference's own parallel-vs-sequential spread, for scale
            extra["rel_diff_ref_parallel_vs_sequential"] = float(np.max(np.abs(out - ref_par)) / np.max(np.abs(out)))
        extra["step_backward_error"] = step_backward_error(out, L, y0, a.T, p, N, m, a.method)
        print(json.dumps({**extra, "impl": "reference", "fn": "solve_ivp_parallel" if parallel else "solve_ivp_sequential",
                          "metric": "ivp_steps_per_s", "value": p * N / t, "ms": t * 1e3,
                          "cores": ncores if parallel else 1, "rel_diff_vs_ours": d, "config": cfg}))


if __name__ == "__main__":
    main()
