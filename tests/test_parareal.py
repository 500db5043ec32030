"""Host pieces of Parareal (include/parsol/parareal.hpp) on the CPU:
matrix_exponential against the unmodified reference (src/parareal.cpp:122-158)
and the SPEC oracles (expm(L, 0) = I, diagonal L, 30-term Taylor series)."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libs():
    from paper_0912_3678_b200 import build
    build.build(verbose=False)
    ours = C.CDLL(os.path.join(ROOT, "paper_0912_3678_b200", "libparsol_b200.so"))
    ref = O.ref() if O.ref_available() else None
    return ours, ref


def expm(lib, fn, L, t):
    m = L.shape[0]
    out = np.zeros((m, m))
    err = C.create_string_buffer(256)
    rc = getattr(lib, fn)(C.c_int(m), np.ascontiguousarray(L).ctypes.data_as(C.c_void_p), C.c_double(t),
                          out.ctypes.data_as(C.c_void_p), err, C.c_size_t(256))
    return rc, out, err.value.decode()


def taylor(A, terms=30):
    out, term = np.eye(A.shape[0]), np.eye(A.shape[0])
    for k in range(1, terms):
        term = term @ A / k
        out = out + term
    return out


def test_expm_spec_examples(libs):
    ours, _ = libs
    rc, E, _ = expm(ours, "psg_expm", np.array([[1.0, 2.0], [3.0, 4.0]]), 0.0)
    assert rc == 0 and np.array_equal(E, np.eye(2))
    rc, E, _ = expm(ours, "psg_expm", np.diag([0.3, -1.7]), 2.0)
    assert abs(E[0, 0] - math.exp(0.6)) <= 1e-14 * math.exp(0.6) and abs(E[1, 1] - math.exp(-3.4)) <= 1e-14
    assert E[0, 1] == 0.0 and E[1, 0] == 0.0
    rng = np.random.default_rng(3)
    for _ in range(5):
        A = rng.uniform(-1, 1, (3, 3))
        A *= 0.9 / np.max(np.sum(np.abs(A), axis=1))  # ||tL|| <= 1 with t = 1/0.9... scaled below
        rc, E, _ = expm(ours, "psg_expm", A, 1.0)
        assert np.max(np.abs(E - taylor(A))) <= 1e-12


@pytest.mark.parametrize("m,t", [(1, -0.25), (3, 0.5), (8, 3.0), (32, 1e-3), (5, 40.0)])
def test_expm_matches_reference(libs, m, t):
    ours, ref = libs
    if ref is None:
        pytest.skip("oracle/_ref not built")
    L = np.random.default_rng(m).uniform(-1, 1, (m, m)) - np.eye(m)
    rc, E, _ = expm(ours, "psg_expm", L, t)
    rc2, Er, _ = expm(ref, "ref_expm", L, t)
    assert rc == 0 and rc2 == 0
    assert np.max(np.abs(E - Er)) <= 1e-13 * max(1.0, np.max(np.abs(Er)))


def test_expm_errors(libs):
    ours, _ = libs
    rc, _, err = expm(ours, "psg_expm", np.array([[np.inf]]), 1.0)
    assert rc == 1 + 19 and "non-finite" in err  # ExpmFailure
