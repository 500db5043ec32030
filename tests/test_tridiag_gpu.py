"""GPU parity of the scalar tridiagonal path (BASELINE configs 0/1) against the
oracle (plain-C restatement, bit-identical to the reference) through the C ABI."""
import numpy as np
import pytest

import oracle as O
import paper_0912_3678_b200 as psg

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _solve_gpu(torch, A, p, f, strategy=psg.Strategy.Lu, device=True, **opts):
    if device:
        GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(torch, A.data))
        F = psg.parallel_factor(GA, p, strategy)
        for k, v in opts.items():
            F.set_option(k, v)
        st = psg.SolveStats()
        x = psg.solve(F, _dev(torch, f), st).cpu().numpy()
    else:
        GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, A.data)
        F = psg.parallel_factor(GA, p, strategy)
        for k, v in opts.items():
            F.set_option(k, v)
        st = psg.SolveStats()
        x = psg.solve(F, f, st)
    return x, st, F


@pytest.mark.parametrize("n,p", [(1 << 20, 1024), (5000, 7), (1000, 2), (64, 4), (300, 3)])
def test_config0_family_matches_oracle(cuda, n, p):
    A, f = O.generate_config(0, n, 1)
    want, _ = O.parallel_solve(A, p, f)
    got, st, _ = _solve_gpu(cuda, A, p, f)
    assert O.rel_err(got, want) <= 1e-12
    assert O.residual(A, got, f) <= 1e-13
    assert st.certificate <= 1e-14


def test_config0_host_path_and_exact_mode(cuda):
    A, f = O.generate_config(0, 1 << 16, 1)
    want, _ = O.parallel_solve(A, 64, f)
    got, st, _ = _solve_gpu(cuda, A, 64, f, device=False)
    assert O.rel_err(got, want) <= 1e-12
    got2, st2, _ = _solve_gpu(cuda, A, 64, f, speculative=0)
    assert O.rel_err(got2, want) <= 1e-12
    assert st2.speculative == 0


def test_generator_bit_identical(cuda):
    for cfg, size in [(0, 4096), (2, 300), (3, 5000), (4, 100)]:
        A, f = O.generate_config(cfg, size, 7)
        GA, gf = psg.generate_config(cfg, size, 7)
        assert np.array_equal(GA.data.cpu().numpy(), A.data)
        assert np.array_equal(gf.cpu().numpy(), f)
        if cfg == 4:
            assert np.array_equal(GA.corner.cpu().numpy(), A.corner)


def test_residual_bit_identical(cuda):
    for cfg, size in [(0, 4096), (2, 300), (3, 5000), (4, 100)]:
        A, f = O.generate_config(cfg, size, 3)
        x = O.solve_sequential(A, f) * (1 + 1e-9)
        GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(cuda, A.data),
                                  None if A.corner is None else _dev(cuda, A.corner), A.corner_rows, A.corner_cols)
        r = psg.residual(GA, _dev(cuda, x), _dev(cuda, f))
        assert r == O.residual(A, x, f)


def test_config1_full_size(cuda):
    torch = cuda
    A, f = psg.generate_config(1, 1 << 26, 2)
    F = psg.parallel_factor(A, 65536)
    st = psg.SolveStats()
    x = psg.solve(F, f, st)
    assert st.speculative == 1 and st.fallbacks == 0
    assert psg.residual(A, x, f) <= 1e-13
    # separator values against the reference-order sequential oracle on a slice is not
    # possible; compare the full solution with the oracle's solve_sequential on host.
    Ah = O.Matrix(A.kind, A.n, A.m, A.s, A.r, A.data.cpu().numpy())
    want = O.solve_sequential(Ah, f.cpu().numpy())
    assert O.rel_err(x.cpu().numpy(), want) <= 1e-12


def _toeplitz(n, lo, d, up):
    data = np.concatenate([np.full(n - 1, lo), np.full(n, d), np.full(n - 1, up)])
    return O.Matrix(O.BANDED, n, 1, 1, 1, data)


def test_weak_dominance_falls_back_to_exact(cuda):
    # rho ~ 0.9: a 32-row truncation is far from exact -> certificate rejects it
    n, p = 40000, 40
    A = _toeplitz(n, -1.0, 2.02, -1.0)
    f = np.sin(np.arange(n) * 0.37)
    want, _ = O.parallel_solve(A, p, f)
    got, st, _ = _solve_gpu(cuda, A, p, f)
    assert st.fallbacks == 1 and st.speculative == 0
    assert O.rel_err(got, want) <= 1e-10
    assert O.residual(A, got, f) <= 1e-13


@pytest.mark.parametrize("n,p", [(20000, 3), (9, 2), (3, 2), (200, 10), (5000, 100)])
def test_refined_and_small_segments(cuda, n, p):
    A, f = O.generate_config(0, n, 5)
    want, _ = O.parallel_solve(A, p, f)
    got, st, _ = _solve_gpu(cuda, A, p, f)
    assert O.rel_err(got, want) <= 1e-12
    assert O.residual(A, got, f) <= 1e-13


def test_toeplitz_known_answer(cuda):
    # Toeplitz(-1,2,-1), n=3, p=2, f=[1,1,1] -> x=[1.5,2,1.5]
    A = _toeplitz(3, -1.0, 2.0, -1.0)
    got, _, _ = _solve_gpu(cuda, A, 2, np.ones(3))
    assert np.allclose(got, [1.5, 2.0, 1.5], rtol=0, atol=1e-15)


def test_reduced_matrix_matches_reference_T(cuda):
    A, f = O.generate_config(0, 1 << 14, 9)
    p = 16
    info = O.factor_info(A, p)
    T = info["T"]
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(cuda, A.data))
    F = psg.parallel_factor(GA, p)
    sub, diag, sup = F.reduced_blocks()
    q = info["dim"]
    assert F.q == q == p - 1
    scale = np.max(np.abs(np.diag(T)))
    assert np.max(np.abs(diag - np.diag(T))) <= 1e-14 * scale
    assert np.max(np.abs(sub[1:] - np.diag(T, -1))) <= 1e-14 * scale
    assert np.max(np.abs(sup[:-1] - np.diag(T, 1))) <= 1e-14 * scale
    # solve_reduced (exact) against a dense solve of the reference T
    rhs = np.cos(np.arange(q))
    xr = psg.solve_reduced(F, rhs)
    assert O.rel_err(xr, np.linalg.solve(T, rhs)) <= 1e-12


def test_strategies_and_errors(cuda):
    A, f = O.generate_config(0, 4096, 4)
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(cuda, A.data))
    want, _ = O.parallel_solve(A, 8, f)
    for s in (psg.Strategy.Lu, psg.Strategy.Lud, psg.Strategy.CyclicReduction, psg.Strategy.LuPivot, psg.Strategy.Qr):
        F = psg.parallel_factor(GA, 8, s)
        got = psg.solve(F, _dev(cuda, f)).cpu().numpy()
        assert O.rel_err(got, want) <= 1e-12
    for s, code in ((psg.Strategy.Arce, psg.Errc.UnsupportedKind),):
        with pytest.raises(psg.Error) as ei:
            psg.parallel_factor(GA, 8, s)
        assert ei.value.code == code
    with pytest.raises(psg.Error) as ei:
        psg.parallel_factor(GA, 1)
    assert ei.value.code == psg.Errc.TooManyPartitions
    with pytest.raises(psg.Error) as ei:
        psg.parallel_factor(GA, 4000)
    assert ei.value.code == psg.Errc.TooManyPartitions


def test_zero_pivot_reports_partition(cuda):
    # p = 3 on n = 3000: bodies [0,1000) [1001,2000) [2001,3000), separators 1000, 2000.
    # Rows 1001/1002 of partition 2 become the [[0,1],[1,0]] block of
    # tests/test_localfact.cpp:369-385 -> ZeroPivot tagged with partition 2.
    n, p = 3000, 3
    A = _toeplitz(n, 1.0, 4.0, 1.0)
    d = A.data.copy()
    sub, dia, sup = 0, n - 1, 2 * n - 1    # a_r = d[sub + r - 1], b_r = d[dia + r], c_r = d[sup + r]
    d[dia + 1001] = 0.0
    d[dia + 1002] = 0.0
    d[sup + 1001] = 1.0
    d[sub + 1002 - 1] = 1.0
    A = O.Matrix(O.BANDED, n, 1, 1, 1, d)
    with pytest.raises(O.OracleError) as eo:
        O.parallel_solve(A, p, np.ones(n))
    assert eo.value.errc == psg.Errc.ZeroPivot and "partition 2" in str(eo.value)
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(cuda, A.data))
    F = psg.parallel_factor(GA, p)
    with pytest.raises(psg.Error) as ei:
        psg.solve(F, _dev(cuda, np.ones(n)))
    assert ei.value.code == psg.Errc.ZeroPivot
    assert "partition 2" in str(ei.value)


import glob as _glob
import os as _os

_GOLD = sorted(_glob.glob(_os.path.join(_os.path.dirname(__file__), "golden", "cfg[01]_*.npz")))


@pytest.mark.parametrize("path", _GOLD, ids=[_os.path.basename(c)[:-4] for c in _GOLD])
def test_cuda_matches_reference_golden(cuda, path):
    g = np.load(path)
    A, f = O.generate_config(int(g["cfg"]), int(g["size"]), int(g["seed"]))
    got, st, F = _solve_gpu(cuda, A, int(g["p"]), f)
    assert O.rel_err(got, g["x"]) <= 1e-12        # vs reference parallel_factor+solve
    assert O.rel_err(got, g["x_seq"]) <= 1e-12    # vs reference solve_sequential
    assert O.residual(A, got, f) <= 1e-13
    assert F.q == int(g["q"]) and F.dim == int(g["dim"])


def test_async_and_refactor(cuda):
    torch = cuda
    A, f = psg.generate_config(1, 1 << 20, 3)
    F = psg.parallel_factor(A, 1024)
    xs = [torch.empty_like(f) for _ in range(3)]
    fs = [f, f * 2.0, torch.flip(f, [0]).contiguous()]
    for fi, xi in zip(fs, xs):
        F.solve_async(fi, xi, timing=True)
    st = psg.SolveStats()
    F.sync(st)
    assert st.speculative == 1 and st.fallbacks == 0 and st.phase3_seconds > 0
    for fi, xi in zip(fs, xs):
        assert psg.residual(A, xi, fi) <= 1e-13
    # new values, same structure: refactor in place
    A2, f2 = psg.generate_config(1, 1 << 20, 4)
    F.refactor(A2)
    x2 = torch.empty_like(f2)
    F.solve_async(f2, x2)
    F.sync()
    assert psg.residual(A2, x2, f2) <= 1e-13
    Ah = O.Matrix(A2.kind, A2.n, 1, 1, 1, A2.data.cpu().numpy())
    assert O.rel_err(x2.cpu().numpy(), O.solve_sequential(Ah, f2.cpu().numpy())) <= 1e-12


def test_async_repairs_failed_speculation(cuda):
    torch = cuda
    n, p = 40000, 40
    A = _toeplitz(n, -1.0, 2.02, -1.0)   # weak dominance: the 32-row truncation is rejected
    f = np.sin(np.arange(n) * 0.37)
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(cuda, A.data))
    F = psg.parallel_factor(GA, p)
    fd = _dev(cuda, f)
    x = torch.empty_like(fd)
    F.solve_async(fd, x)
    st = psg.SolveStats()
    F.sync(st)
    assert st.fallbacks == 1
    want, _ = O.parallel_solve(A, p, f)
    assert O.rel_err(x.cpu().numpy(), want) <= 1e-10


def test_large_n_64bit_offsets(cuda):
    """Maximum sizes: n = 2^28 + 12345 (byte offsets beyond 2^31 in every
    array; ragged bodies), speculative path, certified, residual <= 1e-13."""
    torch = cuda
    n = (1 << 28) + 12345
    A, f = psg.generate_config(1, n, 11)
    F = psg.parallel_factor(A, 1 << 18)
    st = psg.SolveStats()
    x = psg.solve(F, f, st)
    assert st.speculative == 1 and st.certificate <= 1e-14
    assert psg.residual(A, x, f) <= 1e-13
    # spot rows near the end against the row equations directly (host, exact arithmetic on fp64 values)
    d = A.data
    for r in (n - 1, n - 2, (1 << 28) - 7, 1 << 27):
        a = d[r - 1].item() if r > 0 else 0.0
        b = d[n - 1 + r].item()
        c = d[2 * n - 1 + r].item() if r < n - 1 else 0.0
        xm = x[r - 1].item() if r > 0 else 0.0
        xp = x[r + 1].item() if r < n - 1 else 0.0
        lhs = a * xm + b * x[r].item() + c * xp
        assert abs(lhs - f[r].item()) <= 1e-12 * (abs(a * xm) + abs(b * x[r].item()) + abs(c * xp) + abs(f[r].item()))
    del A, f, x, F
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,p", [((1 << 22) + 12345, 4096), (1 << 23, 1024), ((1 << 22) + 7, 2)])
def test_host_buffer_pipeline(cuda, n, p):
    """Host f / x without stats: f arrives in row chunks, x leaves per chunk
    while later chunks still arrive (psg_solve's pipelined host path).  Same
    result, bit for bit, as the device-resident solve."""
    A, f = O.generate_config(0, n, 21)
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(cuda, A.data))
    F = psg.parallel_factor(GA, p)
    x_host = psg.solve(F, f)            # numpy in -> numpy out, pipelined
    x_dev = psg.solve(F, _dev(cuda, f)).cpu().numpy()
    assert np.array_equal(x_host, x_dev)
    want = O.solve_sequential(A, f)
    assert O.rel_err(x_host, want) <= 1e-12
    assert O.residual(A, x_host, f) <= 1e-13


def test_host_buffer_pipeline_fallback(cuda):
    # weak dominance through the pipelined host path: certificate rejects, exact re-solve
    n, p = (1 << 22) + 3, 512
    A = _toeplitz(n, -1.0, 2.02, -1.0)
    f = np.sin(np.arange(n) * 0.37)
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(cuda, A.data))
    F = psg.parallel_factor(GA, p)
    x = psg.solve(F, f)
    assert O.residual(A, x, f) <= 1e-13
    st = psg.SolveStats()
    x2 = psg.solve(F, _dev(cuda, f), st).cpu().numpy()  # the handle stays exact
    assert st.speculative == 0
    assert O.rel_err(x, x2) <= 1e-12


def _planted_unstable(torch, n, p, body, offset):
    """Config-0 distribution with one body made unstable for the no-pivot
    elimination: a 2x2 block [[eps, 1], [1, 1]] (a_r = 0, b_r = 1e-12) deep
    inside body `body`, far from both separators."""
    A, f = O.generate_config(0, n, 5)
    d = A.data.copy()
    plan = O.RefMatrix(A).plan(p) if O.ref_available() else None
    b0 = plan["body"][body][0] if plan else body * (n // p)
    r = b0 + offset
    d[r - 1] = 0.0           # a_r (sub-diagonal of row r)
    d[n - 1 + r] = 1e-12     # b_r
    d[2 * n - 1 + r] = 1.0   # c_r
    d[r] = 1.0               # a_{r+1}
    d[n - 1 + r + 1] = 1.0   # b_{r+1}
    A2 = O.Matrix(A.kind, A.n, A.m, A.s, A.r, d)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    return A2, f, psg.StructuredMatrix(A2.kind, A2.n, A2.m, A2.s, A2.r, dev(d)), dev(f)


def test_body_certificate_catches_planted_instability(cuda):
    """The separator-row certificate cannot see an inaccurate body solve; with
    PSG_OPT_BODY_CERT the certificate covers every body row (componentwise
    backward error from the rows K3 already holds) and rejects it."""
    torch = cuda
    n, p = 1 << 16, 64
    A, f, GA, df = _planted_unstable(torch, n, p, body=10, offset=33 * 3 + 10)
    F = psg.parallel_factor(GA, p)
    st = psg.SolveStats()
    x = psg.solve(F, df, st)
    sep_only = st.certificate
    res_sep_only = psg.residual(GA, x, df)
    F2 = psg.parallel_factor(GA, p)
    F2.set_option("body_cert", 1)
    st2 = psg.SolveStats()
    x2 = psg.solve(F2, df, st2)
    from conftest import record_parity
    record_parity("planted_unstable_body", {"separator_certificate": sep_only, "residual": res_sep_only,
                                            "body_certificate": st2.certificate, "fallbacks": st2.fallbacks})
    assert sep_only <= 1e-14 and res_sep_only > 1e-10  # the separator rows alone pass a wrong solution
    assert st2.certificate > 1e-14                      # the body certificate catches it
    assert st2.fallbacks == 1                           # and the speculative result is re-solved exactly


def test_body_certificate_passes_dominant_systems(cuda):
    torch = cuda
    A, f = psg.generate_config(0, 1 << 20, 1)
    F = psg.parallel_factor(A, 1024)
    F.set_option("body_cert", 1)
    st = psg.SolveStats()
    x = psg.solve(F, f, st)
    assert st.speculative == 1 and st.fallbacks == 0
    assert st.certificate <= 1e-15
    assert psg.residual(A, x, f) <= 1e-13


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_refined_plan_reduced_system_matches_reference(cuda):
    """Bodies longer than one K3 warp (small p) are refined internally; the
    ReducedSystem the API reports is still the reference plan's (built from
    the generic exact path): T, solve_reduced and the reduced rhs against the
    unmodified reference."""
    torch = cuda
    n, p = 70001, 16
    A, f = O.generate_config(0, n, 7)
    R = O.RefMatrix(A)
    RF = R.factor(p)
    Tr = RF.T()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, dev(A.data))
    F = psg.parallel_factor(GA, p)
    assert F.q == Tr.shape[0] == p - 1
    Tg = F.reduced_dense()
    assert np.max(np.abs(Tg - Tr)) <= 1e-14 * np.max(np.abs(Tr))
    rhs = O.random_vector(p - 1, 3)
    xr = psg.solve_reduced(F, rhs)
    assert O.rel_err(xr, np.linalg.solve(Tr, rhs)) <= 1e-13
    x = psg.solve(F, dev(f)).cpu().numpy()
    want, _, _ = RF.solve(f)
    assert O.rel_err(x, want) <= 1e-12
