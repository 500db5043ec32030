"""GPU parity of the K x K block speculative path (blk_kernels.cuh):
BlockTridiagonal m = 2..4 and Banded with max(s, r) = 2..4, bodies long enough
for the truncated interface (>= 16 block rows), against the oracle (bit-
identical to the reference).  Checks that the speculative path was actually
taken (stats.speculative == 1), that it falls back to the exact path when the
certificate fails, and the async API on block kinds."""
import numpy as np
import pytest

import oracle as O
import paper_0912_3678_b200 as psg

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _factor(torch, A, p):
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(torch, A.data), None, 0, 0)
    return psg.parallel_factor(GA, p), GA


SPEC_SHAPES = [  # kind, n, m, s, r, p  (bodies >= 16 K rows; some > 32 M blocks -> refined)
    (1, 4 * 4096, 4, 1, 1, 16),
    (1, 4 * 1000, 4, 1, 1, 7),
    (1, 3 * 3000, 3, 1, 1, 9),
    (1, 2 * 5000, 2, 1, 1, 5),
    (0, 20000, 1, 3, 3, 8),
    (0, 9001, 1, 2, 3, 5),
    (0, 7000, 1, 2, 2, 6),
    (0, 12000, 1, 4, 4, 10),
    (0, 8000, 1, 1, 4, 4),
]


@pytest.mark.parametrize("kind,n,m,s,r,p", SPEC_SHAPES)
def test_block_spec_matches_oracle(cuda, kind, n, m, s, r, p):
    """Dominance 4: the interface decays well inside the truncation window,
    so the certified speculative answer must be the one returned."""
    A = O.generate_random(kind, n, m, s, r, 31 + n, 4.0)
    f = O.random_vector(n, 5)
    want, _ = O.parallel_solve(A, p, f)
    F, GA = _factor(cuda, A, p)
    st = psg.SolveStats()
    x = psg.solve(F, _dev(cuda, f), st).cpu().numpy()
    assert st.speculative == 1, "block speculative path not taken"
    assert st.certificate <= 1e-14
    assert O.rel_err(x, want) <= 1e-12
    assert O.residual(A, x, f) <= 1e-13


@pytest.mark.parametrize("kind,n,m,s,r,p", SPEC_SHAPES)
def test_block_spec_or_fallback_matches_oracle(cuda, kind, n, m, s, r, p):
    """Dominance 2: some shapes decay too slowly for the window; either the
    certificate accepts (omega <= 1e-14) or the exact path answers."""
    A = O.generate_random(kind, n, m, s, r, 31 + n, 2.0)
    f = O.random_vector(n, 5)
    want, _ = O.parallel_solve(A, p, f)
    F, GA = _factor(cuda, A, p)
    st = psg.SolveStats()
    x = psg.solve(F, _dev(cuda, f), st).cpu().numpy()
    assert st.speculative == 1 or st.fallbacks == 1
    if st.speculative:
        assert st.certificate <= 1e-14
    assert O.rel_err(x, want) <= 1e-12
    assert O.residual(A, x, f) <= 1e-13


def test_block_spec_fallback_on_weak_dominance(cuda):
    """Weak dominance: the interface decays too slowly for 16 block rows, the
    certificate fails and the exact path answers."""
    n, m, p = 4 * 2048, 4, 8
    A = O.generate_random(1, n, m, 1, 1, 77, 1.02)
    f = O.random_vector(n, 6)
    want, _ = O.parallel_solve(A, p, f)
    F, _ = _factor(cuda, A, p)
    st = psg.SolveStats()
    x = psg.solve(F, _dev(cuda, f), st).cpu().numpy()
    assert O.rel_err(x, want) <= 1e-10
    if st.speculative == 0:
        assert st.fallbacks >= 1


def test_block_spec_async_and_refactor(cuda):
    torch = cuda
    n, m, p = 4 * 4096, 4, 16
    A1 = O.generate_random(1, n, m, 1, 1, 5, 2.0)
    A2 = O.generate_random(1, n, m, 1, 1, 6, 2.0)
    fs = [O.random_vector(n, 10 + i) for i in range(3)]
    F, GA = _factor(torch, A1, p)
    xs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in fs]
    dfs = [_dev(torch, f) for f in fs]
    for df, dx in zip(dfs, xs):
        F.solve_async(df, dx)
    st = psg.SolveStats()
    F.sync(st)
    for f, dx in zip(fs, xs):
        want, _ = O.parallel_solve(A1, p, f)
        assert O.rel_err(dx.cpu().numpy(), want) <= 1e-12
    GA.data.copy_(_dev(torch, A2.data))
    F.refactor(GA)
    x = psg.solve(F, dfs[0]).cpu().numpy()
    want, _ = O.parallel_solve(A2, p, fs[0])
    assert O.rel_err(x, want) <= 1e-12


def test_block_spec_exact_option_matches(cuda):
    n, m, p = 4 * 4096, 4, 16
    A = O.generate_random(1, n, m, 1, 1, 9, 2.0)
    f = O.random_vector(n, 2)
    F, _ = _factor(cuda, A, p)
    F.set_option("speculative", 0.0)
    st = psg.SolveStats()
    x = psg.solve(F, _dev(cuda, f), st).cpu().numpy()
    assert st.speculative == 0
    want, _ = O.parallel_solve(A, p, f)
    assert O.rel_err(x, want) <= 1e-12
