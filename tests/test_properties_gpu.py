"""SPEC invariants of the solve path on the GPU (reference SPEC.md "Operations"
examples and "Invariants & Properties"): solver equivalence against a dense
solve on many small dominant instances of every kind, the random BABD n=64
p=4 case, residual examples, scheduling determinism (bit-identical repeats,
async == blocking), and the sequential-fraction law (phase-2 operation count
depends on q only)."""
import numpy as np
import pytest

import oracle as O
import paper_0912_3678_b200 as psg

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _gpu_matrix(torch, A):
    return psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, _dev(torch, A.data), _dev(torch, A.corner),
                                A.corner_rows, A.corner_cols)


def _dense(A):
    n = A.n
    D = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        D[:, j] = O.matvec(A, e)
    return D


def _cases():
    rng = np.random.default_rng(2024)
    shapes = [(0, 1, 1, 1), (0, 1, 2, 1), (0, 1, 3, 3), (0, 1, 1, 4), (1, 2, 1, 1), (1, 3, 1, 1), (1, 4, 1, 1),
              (2, 4, 2, 2), (2, 3, 1, 2), (3, 2, 1, 1), (3, 4, 2, 2)]
    out = []
    for t in range(66):
        kind, m, s, r = shapes[t % len(shapes)]
        p = int(rng.integers(2, 6))
        blocks = int(rng.integers(6 * p, 14 * p))
        n = blocks * m if kind else int(rng.integers(8 * p * max(s, r), 30 * p * max(s, r)))
        out.append((kind, n, m, s, r, p, 1000 + t))
    return out


@pytest.mark.parametrize("kind,n,m,s,r,p,seed", _cases())
def test_solver_equivalence_dense(cuda, kind, n, m, s, r, p, seed):
    """SPEC: solve matches a dense-LU oracle <= 1e-10 on dominant random instances (all kinds)."""
    A = O.generate_random(kind, n, m, s, r, seed, 2.0)
    f = O.random_vector(n, seed + 1)
    F = psg.parallel_factor(_gpu_matrix(cuda, A), p)
    x = psg.solve(F, _dev(cuda, f)).cpu().numpy()
    want = np.linalg.solve(_dense(A), f)
    assert O.rel_err(x, want) <= 1e-10
    assert O.residual(A, x, f) <= 1e-13


def test_random_babd_n64_p4(cuda):
    """SPEC: random BABD n=64, p=4 -> matches dense solve <= 1e-10."""
    A = O.generate_random(3, 64, 4, 2, 2, 64, 2.0)
    f = O.random_vector(64, 4)
    F = psg.parallel_factor(_gpu_matrix(cuda, A), 4)
    x = psg.solve(F, _dev(cuda, f)).cpu().numpy()
    assert O.rel_err(x, np.linalg.solve(_dense(A), f)) <= 1e-10
    assert F.q == 5  # p + 1 separators with the corner


def test_residual_examples(cuda):
    """SPEC residual examples: x = 0, f != 0 -> 1.0; exact solve tiny; a 1e-3
    perturbation lands in the [1e-5, 1e-1] sanity band."""
    torch = cuda
    A = O.generate_random(0, 3000, 1, 1, 1, 9, 2.0)
    f = O.random_vector(3000, 2)
    GA = _gpu_matrix(torch, A)
    df = _dev(torch, f)
    assert psg.residual(GA, torch.zeros_like(df), df) == 1.0
    F = psg.parallel_factor(GA, 8)
    x = psg.solve(F, df)
    assert psg.residual(GA, x, df) <= 1e-13
    xp = x * (1 + 1e-3 * torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, 3000)).cuda())
    assert 1e-5 <= psg.residual(GA, xp, df) <= 1e-1


@pytest.mark.parametrize("cfg,size,p", [(0, 1 << 16, 64), (2, 1 << 12, 64), (3, 1 << 16, 128), (4, 1 << 12, 64)])
def test_scheduling_determinism(cuda, cfg, size, p):
    """SPEC: output bit-identical across runs / launch paths (blocking, async, new handle)."""
    torch = cuda
    A, f = psg.generate_config(cfg, size, 5)
    F1 = psg.parallel_factor(A, p)
    x1 = psg.solve(F1, f)
    x2 = psg.solve(F1, f)
    x3 = torch.empty_like(f)
    F1.solve_async(f, x3)
    F1.sync()
    F2 = psg.parallel_factor(A, p)
    x4 = psg.solve(F2, f)
    for other in (x2, x3, x4):
        assert torch.equal(x1, other)


def test_sequential_fraction_law(cuda):
    """SPEC: the phase-2 operation counter depends on q only (exact path, fixed p, varying n)."""
    torch = cuda
    ops = []
    for n in (4000, 8000, 16000):
        A = O.generate_random(0, n, 1, 1, 1, n, 2.0)
        F = psg.parallel_factor(_gpu_matrix(torch, A), 8)
        F.set_option("speculative", 0.0)
        st = psg.SolveStats()
        psg.solve(F, _dev(torch, O.random_vector(n, 1)), st)
        ops.append(st.reduced_ops)
    assert ops[0] == ops[1] == ops[2] > 0
