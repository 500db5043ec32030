"""Per-partition local factorizations on the GPU (psg_local_*, the
reference's LocalFactorization, proj/include/parsol/localfact.hpp:24-125)
against the UNMODIFIED reference (oracle/_ref) on the same blocks:
every field -- fac / dvec, fill-ins z w y v, alpha1 alpha2 beta gamma, kept,
the cyclic-reduction eliminations, the LuPivot / Qr frames, pivot orders and
adaptive extras -- and every member operation (condense, backsolve,
apply_N_inv, apply_S_inv) must be bit-identical (src/localfact.cpp:84-875).
Also solve_reduced on an explicit T (psg_dense_solve vs src/parfact.cpp:134-184)."""
import numpy as np
import pytest

import oracle as O
import paper_0912_3678_b200 as psg

pytestmark = pytest.mark.gpu

LU, LUD, CR, LUPIVOT, QR = 0, 1, 2, 4, 5

# kind, n, m, s, r, p, dominance
MATS = [
    (0, 34, 1, 2, 3, 3, 2.0), (0, 30, 1, 1, 1, 3, 2.0), (0, 23, 1, 1, 1, 3, 2.0), (0, 31, 1, 2, 2, 3, 2.0),
    (0, 400, 1, 1, 1, 4, 2.0), (0, 257, 1, 3, 3, 5, 2.0), (0, 120, 1, 2, 1, 4, 0.3),
    (1, 36, 3, 1, 1, 3, 2.0), (1, 96, 4, 1, 1, 4, 2.0), (1, 64, 2, 1, 1, 4, 0.4),
    (2, 64, 2, 1, 1, 3, 2.0), (2, 120, 4, 2, 2, 3, 2.0),
    (3, 60, 3, 2, 1, 3, 2.0), (3, 96, 4, 2, 2, 4, 0.5),
]


def _block(kind, n, m, s, r, p, dom, i):
    data, corner = O.ref_generate_random(kind, n, m, s, r, 1000 + n + 7 * s + r, dom)
    A = O.Matrix(kind, n, m, s, r, data, corner, m if kind == 3 else 0, m if kind == 3 else 0)
    return O.ref_extract_block(A, p, i)


def _psg_block(b):
    return psg.PartitionBlock(b["kind"], b["m"], b["s"], b["r"], b["L"], b["k0"], b["k1"], b["env_s"], b["env_r"],
                              b["env"], b["b0"], b["c0"], b["b1"], b["c1"], b["a_right"])


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64 if np.asarray(a).dtype == np.float64 else np.uint32).ravel()


def _same(got, want, what):
    got, want = np.ascontiguousarray(got).ravel(), np.ascontiguousarray(want).ravel()
    assert got.shape == want.shape, f"{what}: shape {got.shape} vs {want.shape}"
    assert np.array_equal(_bits(got), _bits(want)), \
        f"{what}: max |diff| {np.max(np.abs(got.astype(float) - want.astype(float))) if got.size else 0}"


FIELDS = {"fac": 0, "dvec": 1, "z": 2, "w": 3, "y": 4, "v": 5, "alpha1": 6, "alpha2": 7, "beta": 8, "gamma": 9,
          "kept": 10, "cr_elim_idx": 11, "cr_elim_mat": 12, "cr_d2": 13, "cr_d2inv": 14, "cr_cmat": 15,
          "cr_rmat_d2inv": 16, "wmid": 17, "lmat": 18, "linv": 19, "a_order": 20, "kept_rows": 21,
          "kept_cols": 22, "extra_pos": 23, "extra_alpha": 24}
INT_FIELDS = {"cr_elim_idx", "a_order", "kept_rows", "kept_cols", "extra_pos"}


def _compare(b, strategy, tol=1e-8):
    try:
        want = O.RefLocal(b, strategy, tol)
    except O.OracleError as e:
        with pytest.raises(psg.Error) as ei:
            psg.factor(strategy, _psg_block(b), tol)
        assert int(ei.value.code) == e.errc
        return None
    got = psg.factor(strategy, _psg_block(b), tol)
    assert got.kept_dim == want.kept_dim
    assert got.cr_levels == want.cr_levels
    assert got.info["n_extras"] == want.n_extras
    big = max(want.dim * want.dim, 5 * want.n_elims * max(want.g, 1) ** 2, 3 * want.dim, 64)
    for name, fid in FIELDS.items():
        dt = np.int32 if name in INT_FIELDS else np.float64
        w = want.field(fid, big, dt)
        g = got.read(name, w.size, dt) if w.size else np.zeros(0, dt)
        _same(g, w, f"strategy {strategy} field {name}")
    rng = np.random.default_rng(b["L"] * 31 + strategy)
    f = rng.uniform(-1, 1, b["L"])
    gh, kr = got.condense(f)
    wgh, wkr = want.op(0, f)
    _same(gh, wgh, "condense ghat")
    _same(kr, wkr, "condense kept_rhs")
    xk = rng.uniform(-1, 1, want.kept_dim)
    _same(got.backsolve(gh, xk), want.op(1, wgh, xk), "backsolve")
    _same(got.apply_N_inv(f), want.op(2, f), "apply_N_inv")
    _same(got.apply_S_inv(f), want.op(3, f), "apply_S_inv")
    return got


@pytest.mark.parametrize("kind,n,m,s,r,p,dom", MATS)
def test_local_factor_bit_identical(cuda, kind, n, m, s, r, p, dom):
    for i in sorted({1, 2, p}):
        b = _block(kind, n, m, s, r, p, dom, i)
        for strategy in (LU, LUD, LUPIVOT, QR):
            _compare(b, strategy)
        if kind == 1 or (kind == 0 and s == 1 and r == 1):
            _compare(b, CR)


def test_local_factor_triggers_extras_like_reference(cuda):
    """Non-dominant bodies: LuPivot / Qr defer pivots into adaptive extras
    exactly where the reference does (tests/test_localfact.cpp:263-297)."""
    body = np.zeros((5, 5))
    body[0, 0], body[0, 1], body[1, 0], body[1, 1], body[1, 2] = 2, 1, 1, 0.5, 1
    body[2, 2], body[2, 3], body[3, 2], body[3, 3], body[3, 4], body[4, 3], body[4, 4] = 3, 1, 1, 3, 1, 1, 3
    L = 5
    env = np.zeros((L, 2 * L - 1))
    for i in range(L):
        for j in range(L):
            env[i, j - i + L - 1] = body[i, j]
    e = lambda row: (np.arange(L) == row).astype(float)  # noqa: E731
    b = dict(kind=0, m=1, s=1, r=1, L=L, k0=1, k1=1, env_s=L - 1, env_r=L - 1, env=env.ravel(),
             b0=e(0), c0=e(0), b1=e(4), c1=e(4), a_right=np.array([3.0]))
    for strategy in (LUPIVOT, QR):
        got = _compare(b, strategy)
        assert got.info["n_extras"] == 1
        assert list(got.field("extra_pos")) == [1]


def test_zero_pivot_and_errors_match_reference(cuda):
    L = 2  # body [[0,1],[1,0]] (tests/test_localfact.cpp:369-385), envelope rows [a b c]
    b = dict(kind=0, m=1, s=1, r=1, L=L, k0=1, k1=1, env_s=1, env_r=1, env=np.array([0.0, 0.0, 1.0, 1.0, 0.0, 0.0]),
             b0=np.zeros(2), c0=np.zeros(2), b1=np.zeros(2), c1=np.zeros(2), a_right=np.array([1.0]))
    for strategy in (LU, LUD):
        with pytest.raises(psg.Error) as ei:
            psg.factor(strategy, _psg_block(b), 1e-8)
        assert ei.value.code == psg.Errc.ZeroPivot
        with pytest.raises(O.OracleError):
            O.RefLocal(b, strategy)
    _compare(b, LUPIVOT, 1e-10)
    with pytest.raises(psg.Error) as ei:
        psg.factor(LUPIVOT, _psg_block(b), 0.0)
    assert ei.value.code == psg.Errc.InvalidParameter
    blk = _block(0, 30, 1, 2, 1, 3, 2.0, 2)
    with pytest.raises(psg.Error) as ei:
        psg.factor(CR, _psg_block(blk))
    assert ei.value.code == psg.Errc.UnsupportedStructure


@pytest.mark.parametrize("n", [1, 2, 3, 17, 64, 300])
def test_dense_reduced_solve_bit_identical(cuda, n):
    rng = np.random.default_rng(n)
    T = rng.uniform(-1, 1, (n, n)) + np.diag(rng.uniform(-0.5, 0.5, n))
    rhs = rng.uniform(-1, 1, n)
    x, ops = psg.dense_solve(T, rhs)
    wx, wops = O.ref_solve_reduced_dense(T, rhs)
    _same(x, wx, "dense reduced solve")
    assert ops == wops


def test_dense_reduced_solve_hand_cases(cuda):
    """SPEC.md solve_reduced examples: T = I -> x = rhs; [[2,1],[1,2]] x = [3,3] -> [1,1]."""
    x, _ = psg.dense_solve(np.eye(4), np.arange(4.0))
    assert np.array_equal(x, np.arange(4.0))
    x, _ = psg.dense_solve(np.array([[2.0, 1.0], [1.0, 2.0]]), np.array([3.0, 3.0]))
    assert np.allclose(x, [1.0, 1.0], rtol=0, atol=1e-15)
    with pytest.raises(psg.Error) as ei:
        psg.dense_solve(np.zeros((3, 3)), np.ones(3))
    assert ei.value.code == psg.Errc.SingularReducedSystem
