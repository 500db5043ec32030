"""Time-parallel linear IVP solver on the GPU (include/parsol/odeparallel.hpp,
host/host_ode.cpp: the discrete trajectory solved as one BVP-layout BABD by
the chain path) against the UNMODIFIED reference (src/odeparallel.cpp in
oracle/_ref): identical forcing values through one C callback, both methods,
padded dimensions (m = 1, 3, 5), short grids, errors."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GFUN = C.CFUNCTYPE(None, C.c_double, C.POINTER(C.c_double), C.c_void_p)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def libs(cuda):
    from paper_0912_3678_b200 import build
    build.build(verbose=False)
    ours = C.CDLL(os.path.join(ROOT, "paper_0912_3678_b200", "libparsol_b200.so"))
    ours.psg_ode_solve.restype = C.c_int
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = O.ref()
    ref.ref_ode_solve.restype = C.c_int
    return ours, ref


def forcing(m, kind):
    if kind == "none":
        return None
    if kind == "trig":
        def g(t, out, ctx):
            for q in range(m):
                out[q] = math.sin((q + 1) * t) + 0.5 * math.cos(2.0 * t)
    else:  # "step"
        def g(t, out, ctx):
            for q in range(m):
                out[q] = 1.0 if t < 0.5 else -0.25 * q
    return GFUN(g)


def run(lib, fn, m, L, y0, t0, T, p, N, method, g, extra=()):
    out = np.zeros((p * N + 1) * m)
    err = C.create_string_buffer(256)
    args = [C.c_int(m), L.ctypes.data_as(C.c_void_p), y0.ctypes.data_as(C.c_void_p), C.c_double(t0),
            C.c_double(T), C.c_int(p), C.c_int(N), C.c_int(method), g if g is not None else C.cast(None, GFUN),
            C.c_void_p(None)]
    rc = getattr(lib, fn)(*args, *extra, out.ctypes.data_as(C.c_void_p), *([C.byref(C.c_double())] if fn ==
                          "psg_ode_solve" else []), err, C.c_size_t(256))
    return rc, out, err.value.decode()


def problem(kind, m, seed=1):
    rng = np.random.default_rng(seed)
    if kind == "oscillator":
        L = np.array([[0.0, 1.0], [-1.0, 0.0]])
    elif kind == "heat":  # 1-D heat equation, method of lines, Dirichlet ends
        h = 1.0 / (m + 1)
        L = (np.diag(-2.0 * np.ones(m)) + np.diag(np.ones(m - 1), 1) + np.diag(np.ones(m - 1), -1)) / h ** 2
    else:  # random, stable
        L = rng.uniform(-1, 1, (m, m)) - 2.0 * np.eye(m)
    y0 = rng.uniform(-1, 1, m)
    return np.ascontiguousarray(L), y0


CASES = [  # name, kind, m, forcing, T, p, N, method
    ("oscillator-ie", "oscillator", 2, "none", 10.0, 8, 256, 0),
    ("oscillator-trap", "oscillator", 2, "none", 10.0, 8, 256, 1),
    ("random3-trig", "random", 3, "trig", 2.0, 16, 100, 1),
    ("random5-step", "random", 5, "step", 1.0, 12, 80, 0),
    ("random4-trig", "random", 4, "trig", 3.0, 64, 32, 1),
    ("heat8-trap", "heat", 8, "trig", 0.1, 64, 64, 1),
    ("scalar1", "random", 1, "trig", 5.0, 5, 200, 0),
    ("short", "random", 2, "trig", 1.0, 1, 3, 1),
]


@pytest.mark.parametrize("name,kind,m,fk,T,p,N,method", CASES, ids=[c[0] for c in CASES])
def test_ode_matches_reference(libs, name, kind, m, fk, T, p, N, method):
    ours, ref = libs
    L, y0 = problem(kind, m)
    g = forcing(m, fk)
    rc, x, err = run(ours, "psg_ode_solve", m, L, y0, 0.0, T, p, N, method, g)
    assert rc == 0, err
    for parallel in (1, 0):
        rc2, want, err2 = run(ref, "ref_ode_solve", m, L, y0, 0.0, T, p, N, method, g, extra=(C.c_int(parallel),))
        assert rc2 == 0, err2
        assert O.rel_err(x, want) <= 1e-12, (name, parallel, O.rel_err(x, want))
    assert np.array_equal(x[:m], y0)


def test_ode_errors(libs):
    ours, _ = libs
    L, y0 = problem("random", 9)
    rc, _, err = run(ours, "psg_ode_solve", 9, L, y0, 0.0, 1.0, 4, 10, 0, None)
    assert rc == 1 + 9 and "dimension" in err  # UnsupportedStructure
    L, y0 = problem("random", 2)
    rc, _, err = run(ours, "psg_ode_solve", 2, L, y0, 1.0, 1.0, 4, 10, 0, None)
    assert rc == 1 + 18  # InvalidInterval
