"""Parareal on the GPU (include/parsol/parareal.hpp -> psg_pr_*, pr_kernels.cuh)
against the UNMODIFIED reference parareal_solve (oracle/_ref,
src/parareal.cpp:94-120): same forcing through one C callback, same
propagators; iterations equal, inits within 1e-12, histories alike; the
SPEC properties (coarse == fine converges in one iteration, p = 1, iterate
p-1 exact, equivalence with the time-parallel trajectory)."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GFUN = C.CFUNCTYPE(None, C.c_double, C.POINTER(C.c_double), C.c_void_p)
FINE, COARSE, EXPM = 0, 1, 2
IE, TRAP = 0, 1

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def libs(cuda):
    from paper_0912_3678_b200 import build
    build.build(verbose=False)
    ours = C.CDLL(os.path.join(ROOT, "paper_0912_3678_b200", "libparsol_b200.so"))
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    return ours, O.ref()


def heat(m):
    inv = float(m + 1) ** 2
    L = np.diag(-2.0 * inv * np.ones(m)) + np.diag(inv * np.ones(m - 1), 1) + np.diag(inv * np.ones(m - 1), -1)
    y0 = np.sin(np.pi * np.arange(1, m + 1) / (m + 1))
    return np.ascontiguousarray(L), y0


def trig(m):
    def g(t, out, ctx):
        for q in range(m):
            out[q] = math.sin((q + 1) * t) + 0.25
    return GFUN(g)


def run(lib, fn, L, y0, t0, T, p, N, g, fine, coarse, tol=1e-8, max_iter=-1):
    m = len(y0)
    inits = np.zeros(p * m)
    cap = max(2 * p, max_iter, 1)
    hist = np.zeros(cap)
    it, conv = C.c_int(), C.c_int()
    err = C.create_string_buffer(256)
    rc = getattr(lib, fn)(C.c_int(m), L.ctypes.data_as(C.c_void_p), y0.ctypes.data_as(C.c_void_p), C.c_double(t0),
                          C.c_double(T), C.c_int(p), C.c_int(N), g if g is not None else C.cast(None, GFUN),
                          C.c_void_p(None), *[C.c_int(v) for v in fine], *[C.c_int(v) for v in coarse],
                          C.c_double(tol), C.c_int(max_iter), inits.ctypes.data_as(C.c_void_p),
                          hist.ctypes.data_as(C.c_void_p), C.c_int(cap), C.byref(it), C.byref(conv), err,
                          C.c_size_t(256))
    assert rc == 0, err.value
    return inits.reshape(p, m), hist[: it.value], it.value, conv.value


def compare(libs, L, y0, T, p, N, g, fine, coarse, tol=1e-8, max_iter=-1):
    ours, ref = libs
    a = run(ours, "psg_parareal_solve", L, y0, 0.0, T, p, N, g, fine, coarse, tol, max_iter)
    b = run(ref, "ref_parareal_solve", L, y0, 0.0, T, p, N, g, fine, coarse, tol, max_iter)
    assert (a[2], a[3]) == (b[2], b[3])  # iterations, converged
    assert O.rel_err(a[0], b[0]) <= 1e-12, O.rel_err(a[0], b[0])
    scale = np.max(np.abs(b[0]))
    big = b[1] > 1e-6 * scale  # update norms well above rounding agree closely
    assert np.allclose(a[1][big], b[1][big], rtol=1e-8, atol=0)
    return a


CASES = [  # name, problem, m, T, p, N, forcing, fine, coarse
    ("heat32-ie", "heat", 32, 0.1, 8, 100, False, (FINE, IE, 100), (COARSE, IE, 1)),
    ("heat32-trap-expm", "heat", 32, 0.1, 8, 50, False, (FINE, TRAP, 50), (EXPM, IE, 1)),
    ("heat64", "heat", 64, 0.05, 16, 40, False, (FINE, IE, 40), (COARSE, IE, 2)),
    ("random5-forced", "random", 5, 2.0, 12, 60, True, (FINE, TRAP, 60), (COARSE, IE, 1)),
    ("random3-forced-expm", "random", 3, 1.0, 6, 30, True, (FINE, IE, 30), (EXPM, TRAP, 4)),
    ("heat16-many", "heat", 16, 0.2, 64, 20, False, (FINE, IE, 20), (COARSE, IE, 1)),
]


@pytest.mark.parametrize("name,kind,m,T,p,N,forced,fine,coarse", CASES, ids=[c[0] for c in CASES])
def test_parareal_matches_reference(libs, name, kind, m, T, p, N, forced, fine, coarse):
    if kind == "heat":
        L, y0 = heat(m)
    else:
        rng = np.random.default_rng(m)
        L = np.ascontiguousarray(rng.uniform(-1, 1, (m, m)) - 2.0 * np.eye(m))
        y0 = rng.uniform(-1, 1, m)
    compare(libs, L, y0, T, p, N, trig(m) if forced else None, fine, coarse)


def test_coarse_equals_fine_one_iteration(libs):
    L, y0 = heat(8)
    inits, _, it, conv = compare(libs, L, y0, 0.1, 6, 10, None, (FINE, IE, 10), (FINE, IE, 10))
    assert it == 1 and conv == 1


def test_single_window(libs):
    L, y0 = heat(4)
    inits, hist, it, conv = compare(libs, L, y0, 0.1, 1, 10, None, (FINE, IE, 10), (COARSE, IE, 1))
    assert it == 0 and conv == 1 and np.array_equal(inits[0], y0)


def test_not_converged_is_soft(libs):
    L, y0 = heat(16)
    inits, hist, it, conv = compare(libs, L, y0, 0.1, 16, 50, None, (FINE, IE, 50), (COARSE, IE, 1), 1e-14, 2)
    assert it == 2 and conv == 0 and len(hist) == 2


def test_converged_inits_equal_the_time_parallel_trajectory(libs):
    """SPEC invariant: with the fine propagator matching odeparallel's
    method/steps, converged inits equal the window starts of the discrete
    trajectory (solve_ivp_parallel, m <= 8) <= 1e-12."""
    ours, _ = libs
    m, p, N = 8, 8, 100
    L, y0 = heat(m)
    inits, _, _, conv = run(ours, "psg_parareal_solve", L, y0, 0.0, 0.1, p, N, None, (FINE, IE, N), (COARSE, IE, 1),
                            1e-15, 3 * p)
    traj = np.zeros((p * N + 1) * m)
    cert = C.c_double()
    err = C.create_string_buffer(256)
    rc = ours.psg_ode_solve(C.c_int(m), L.ctypes.data_as(C.c_void_p), y0.ctypes.data_as(C.c_void_p), C.c_double(0.0),
                            C.c_double(0.1), C.c_int(p), C.c_int(N), C.c_int(0), C.cast(None, GFUN), C.c_void_p(None),
                            traj.ctypes.data_as(C.c_void_p), C.byref(cert), err, C.c_size_t(256))
    assert rc == 0, err.value
    starts = traj.reshape(p * N + 1, m)[::N][:p]
    assert O.rel_err(inits, starts) <= 1e-12


def test_nilpotency_decay(libs):
    """SPEC example: scalar lambda = -1, p = 4, fine = exact exponential, coarse
    = 1-step implicit Euler: iterate p-1 reproduces the fine sequential values."""
    ours, _ = libs
    L, y0 = np.array([[-1.0]]), np.array([1.0])
    inits, hist, it, _ = run(ours, "psg_parareal_solve", L, y0, 0.0, 1.0, 4, 1, None, (EXPM, IE, 1),
                             (COARSE, IE, 1), 1e-300, 3)
    want = np.exp(-0.25 * np.arange(4))
    assert np.max(np.abs(inits[:, 0] - want)) <= 1e-12
