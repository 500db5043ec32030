"""Pivoting strategies (LuPivot, Qr) with adaptive reduced-system growth, and
the circulant-like kind, on the GPU (csrc/piv_kernels.cuh) against the
UNMODIFIED reference in oracle/_ref (src/localfact.cpp:517-607,
src/parfact.cpp:72-184): reduced layout (q, positions, block sizes) equal,
reduced matrix T bit-identical, solution within 1e-10 (SPEC factor_lu_pivot:
"solve through parfact still matches dense oracle <= 1e-10")."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_0912_3678_b200 as psg

pytestmark = pytest.mark.gpu

LU, LUD, CR, LUPIVOT, QR = 0, 1, 2, 4, 5


def entry_count(kind, n, m, s, r):
    if kind == 4:
        return (s + r + 1) * n
    return int(O.lib().or_body_entry_count(kind, n, m, s, r))


def ref_random(kind, n, m, s, r, seed, dominance):
    data = np.empty(entry_count(kind, n, m, s, r))
    corner = np.empty(m * m) if kind == 3 else None
    err = C.create_string_buffer(256)
    rc = O.ref().ref_generate_random(kind, n, m, s, r, seed, dominance, O._ptr(data), O._ptr(corner), err, 256)
    assert rc == 0, err.value
    cr = m if kind == 3 else 0
    return O.Matrix(kind, n, m, s, r, data, corner, cr, cr)


def ours(torch, A, p, strategy, tol, f):
    dev = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, dev(A.data), dev(A.corner), A.corner_rows, A.corner_cols)
    F = psg.parallel_factor(GA, p, strategy, tol)
    st = psg.SolveStats()
    x = psg.solve(F, dev(f), st).cpu().numpy()
    return F, x, st


def reference(A, p, strategy, tol, f):
    R = O.RefMatrix(A).factor_tol(p, strategy, tol)
    x, ops, _ = R.solve(f)
    pos, size = R.layout()
    return R, x, pos, size, ops


def check_parity(torch, A, p, strategy, tol, seed=3, t_exact=True):
    f = O.random_vector(A.n, seed)
    R, want, rpos, rsize, rops = reference(A, p, strategy, tol, f)
    F, got, st = ours(torch, A, p, strategy, tol, f)
    q, dim = R.dims()
    assert (F.q, F.dim) == (q, dim)
    pos, size = F.reduced_layout()
    assert np.array_equal(pos, rpos) and np.array_equal(size, rsize)
    if dim <= 2048:
        T, Tr = F.reduced_dense(), R.T()
        if t_exact:
            assert np.array_equal(T, Tr), np.max(np.abs(T - Tr))
        else:
            assert np.max(np.abs(T - Tr)) <= 1e-13 * np.max(np.abs(Tr))
    assert O.rel_err(got, want) <= 1e-10, O.rel_err(got, want)
    assert st.reduced_ops == rops
    seps = p + 1 if F.has_corner else p - 1
    return F, got, F.q - seps


CASES = [  # kind, n, m, s, r, p, dominance
    (0, 300, 1, 1, 1, 4, 0.0), (0, 301, 1, 2, 1, 5, 0.0), (0, 400, 1, 3, 3, 4, 0.0),
    (1, 240, 2, 1, 1, 4, 0.0), (1, 360, 3, 1, 1, 5, 0.0), (1, 256, 4, 1, 1, 4, 0.3),
    (2, 400, 4, 2, 2, 5, 0.0), (2, 240, 3, 1, 2, 4, 0.0),
    (3, 240, 2, 1, 1, 4, 0.0), (3, 320, 4, 2, 2, 4, 0.0),
    (4, 300, 1, 1, 1, 4, 0.0), (4, 301, 1, 2, 0, 5, 0.0), (4, 250, 1, 1, 2, 3, 0.0),
]


@pytest.mark.parametrize("strategy", [LUPIVOT, QR], ids=["lupivot", "qr"])
@pytest.mark.parametrize("kind,n,m,s,r,p,dom", CASES)
def test_pivoting_matches_reference(cuda, strategy, kind, n, m, s, r, p, dom):
    A = ref_random(kind, n, m, s, r, 40 + n + kind, dom)
    check_parity(cuda, A, p, strategy, 1e-8)


@pytest.mark.parametrize("strategy", [LUPIVOT, QR], ids=["lupivot", "qr"])
@pytest.mark.parametrize("kind,n,m,s,r,p,tol", [(0, 160, 1, 1, 1, 8, 0.1), (0, 200, 1, 2, 2, 8, 0.08),
                                                (1, 192, 2, 1, 1, 8, 0.08), (4, 160, 1, 1, 1, 8, 0.1),
                                                (3, 192, 2, 1, 1, 6, 0.05)])
def test_adaptive_extras_match_reference(cuda, strategy, kind, n, m, s, r, p, tol):
    """A large tol defers many pivots: the reduced system grows by exactly the
    reference's extras, at the reference's positions."""
    A = ref_random(kind, n, m, s, r, 7 + n, 0.0)
    _, _, extras = check_parity(cuda, A, p, strategy, tol)
    assert extras > 0


def planted_tridiagonal(n=40):
    """Body 2 starts with the rank-1 block [[1,2],[2,4]] and A(23,22) = 0: after
    the first column is eliminated, column 22 vanishes on the active rows."""
    A = ref_random(0, n, 1, 1, 1, 5, 3.0)
    sub, diag, sup = A.data[: n - 1], A.data[n - 1: 2 * n - 1], A.data[2 * n - 1:]
    diag[21], sup[21], sub[21], diag[22], sub[22] = 1.0, 2.0, 2.0, 4.0, 0.0
    return A


@pytest.mark.parametrize("strategy", [LUPIVOT, QR], ids=["lupivot", "qr"])
def test_planted_singular_block_emits_one_extra(cuda, strategy):
    A = planted_tridiagonal()
    F, x, extras = check_parity(cuda, A, 2, strategy, 1e-8)
    assert extras == 1 and F.q == 2  # one separator + one extra (SPEC factor_lu_pivot example)
    pos, size = F.reduced_layout()
    assert list(pos) == [20, 22]
    # backward error on par with the reference's own (the deferred pivot is ~1e-16, not 0, under Qr)
    f = O.random_vector(A.n, 3)
    _, xr, _, _, _ = reference(A, 2, strategy, 1e-8, f)
    assert O.residual(A, x, f) <= max(1e-13, 3 * O.residual(A, xr, f))


@pytest.mark.parametrize("strategy", [LU, LUD])
@pytest.mark.parametrize("kind,n,s,r,p", [(4, 300, 1, 0, 4), (4, 301, 2, 0, 5), (4, 400, 3, 0, 4)])
def test_circulant_no_pivot_matches_reference(cuda, strategy, kind, n, s, r, p):
    """Canonical circulant-like (r = 0); rotated ones (r > 0) break the no-pivot
    factorization in the reference too (SURVEY probe: rel. err 1e70)."""
    A = ref_random(kind, n, 1, s, r, 11 + n, 2.0)
    f = O.random_vector(A.n, 3)
    R, want, rpos, rsize, _ = reference(A, p, strategy, 1e-8, f)
    F, got, _ = ours(cuda, A, p, strategy, 1e-8, f)
    pos, size = F.reduced_layout()
    assert np.array_equal(pos, rpos) and np.array_equal(size, rsize)
    assert O.rel_err(got, want) <= 1e-10


def test_rotated_circulant_needs_pivoting(cuda):
    """SURVEY probe: a rotated circulant (r = 1) with unit dominance loses the
    no-pivot factorization's accuracy; LuPivot / Qr solve it."""
    A = ref_random(4, 256, 1, 1, 1, 77, 1.0)
    f = O.random_vector(A.n, 3)
    dense = np.zeros((A.n, A.n))
    for i in range(A.n):
        for d in range(-A.s, A.r + 1):
            dense[i, (i + d) % A.n] = A.data[(d + A.s) * A.n + i]
    want = np.linalg.solve(dense, f)
    for strategy in (LUPIVOT, QR):
        _, got, _ = ours(cuda, A, 4, strategy, 1e-8, f)
        assert O.rel_err(got, want) <= 1e-10


def test_solve_reduced_matches_dense_T(cuda):
    A = ref_random(0, 160, 1, 1, 1, 9, 0.0)
    F, _, _ = ours(cuda, A, 8, LUPIVOT, 0.1, O.random_vector(160, 1))
    T = F.reduced_dense()
    rhs = np.cos(np.arange(F.dim))
    assert O.rel_err(psg.solve_reduced(F, rhs), np.linalg.solve(T, rhs)) <= 1e-11


def test_errors(cuda):
    A = ref_random(0, 60, 1, 1, 1, 5, 2.0)
    A.data[59:119][20:40] = 0.0  # body 2 (rows 20..39) with a zero diagonal and ...
    A.data[:59][19:39] = 0.0     # ... zero sub-diagonal: every column of the body is deferred
    A.data[119:][20:39] = 0.0
    f = O.random_vector(60, 1)
    with pytest.raises(psg.Error) as e:
        ours(cuda, A, 3, LUPIVOT, 1e-8, f)
    assert e.value.code in (psg.Errc.ExhaustedBody, psg.Errc.UnsupportedStructure)
    with pytest.raises(psg.Error) as e:
        ours(cuda, ref_random(4, 100, 1, 1, 1, 2, 2.0), 4, CR, 1e-8, O.random_vector(100, 1))
    assert e.value.code == psg.Errc.UnsupportedKind


def test_refactor_rebuilds_layout(cuda):
    A = planted_tridiagonal()
    f = O.random_vector(A.n, 3)
    F, _, _ = ours(cuda, A, 2, LUPIVOT, 1e-8, f)
    assert F.q == 2
    B = ref_random(0, A.n, 1, 1, 1, 5, 3.0)  # dominant: no extras
    dev = lambda a: cuda.from_numpy(np.ascontiguousarray(a)).cuda()
    F.refactor(psg.StructuredMatrix(0, B.n, 1, 1, 1, dev(B.data)))
    q = C.c_int()
    psg.lib().psg_reduced_info(F.handle, C.byref(q), None, None, None)
    assert q.value == 1
    x = psg.solve(F, dev(f)).cpu().numpy()
    assert O.residual(B, x, f) <= 1e-13
