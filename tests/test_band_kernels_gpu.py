"""Edge cases of the round-2 kernels of the block kinds, against the oracle
(bit-identical to the reference's parallel_factor + solve):

* band_spec_kernel / band_body_kernel (Banded, scalar band arithmetic): body
  lengths that give every lane layout (odd chunk stride R, short last lane,
  a single lane), s != r, K = 2..4, and weak dominance (the lane-level system
  less decoupled: more Jacobi sweeps, PCR, or the certified fallback);
* blktri_spec_kernel / blktri_body_kernel (BlockTridiagonal, two threads per
  body): odd and small block-row counts per body (the meeting row m = NB / 2),
  and data / rhs not 32-byte aligned (the scalar-load path of the kernels).
"""
import numpy as np
import pytest

import oracle as O
import paper_0912_3678_b200 as psg

pytestmark = pytest.mark.gpu


def _solve(torch, A, p, f, data_offset=0, f_offset=0):
    data = torch.zeros(A.data.size + data_offset, dtype=torch.float64, device="cuda")
    data[data_offset:] = torch.from_numpy(A.data).cuda()
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, data[data_offset:], None, 0, 0)
    fd = torch.zeros(A.n + f_offset, dtype=torch.float64, device="cuda")
    fd[f_offset:] = torch.from_numpy(f).cuda()
    F = psg.parallel_factor(GA, p)
    st = psg.SolveStats()
    x = psg.solve(F, fd[f_offset:], st).cpu().numpy()
    return x, st


# body length L (rows) of the reference plan: n = p (L + K) - K with K = max(s, r);
# neighbouring bodies are merged while the union fits one body kernel (576
# rows), so the kernel sees bodies of about 561 / 500 / 406 / 509 / 575 rows
@pytest.mark.parametrize("L", [48, 61, 97, 200, 509, 575])
@pytest.mark.parametrize("s,r", [(3, 3), (1, 3), (3, 2)])
def test_band_body_lane_layouts(cuda, L, s, r):
    K, p = max(s, r), 24
    n = p * (L + K) - K
    A = O.generate_random(0, n, 1, s, r, 1000 + L + 10 * s + r, 4.0)
    f = O.random_vector(n, L)
    want, _ = O.parallel_solve(A, p, f)
    x, st = _solve(cuda, A, p, f)
    assert st.speculative == 1, "band speculative path not taken"
    assert st.certificate <= 1e-14
    assert O.rel_err(x, want) <= 1e-12
    assert O.residual(A, x, f) <= 1e-13


@pytest.mark.parametrize("s,r,L", [(2, 2, 130), (4, 4, 300), (1, 4, 260), (4, 1, 260)])
def test_band_k2_k4(cuda, s, r, L):
    K, p = max(s, r), 5
    n = p * (L + K) - K
    A = O.generate_random(0, n, 1, s, r, 7 + L, 4.0)
    f = O.random_vector(n, 3)
    want, _ = O.parallel_solve(A, p, f)
    x, st = _solve(cuda, A, p, f)
    assert st.speculative == 1
    assert O.rel_err(x, want) <= 1e-12


@pytest.mark.parametrize("dominance", [1.3, 1.05])
def test_band_weak_dominance(cuda, dominance):
    """Less decoupled lane-level systems (more Jacobi sweeps or PCR) and
    windows that may be too short (certificate -> exact path): the answer
    must match the reference either way."""
    s = r = 3
    L, p = 509, 8
    n = p * (L + 3) - 3
    A = O.generate_random(0, n, 1, s, r, 41, dominance)
    f = O.random_vector(n, 9)
    want, _ = O.parallel_solve(A, p, f)
    x, st = _solve(cuda, A, p, f)
    assert st.speculative == 1 or st.fallbacks >= 1
    assert O.rel_err(x, want) <= 1e-10
    assert O.residual(A, x, f) <= 1e-12


@pytest.mark.parametrize("NB", [16, 17, 33, 64, 65])
def test_blktri_body_meeting_rows(cuda, NB):
    """Two threads per body meet at block row NB / 2: odd and even NB."""
    m, p = 4, 6
    n = m * (p * (NB + 1) - 1)
    A = O.generate_random(1, n, m, 1, 1, 500 + NB, 4.0)
    f = O.random_vector(n, NB)
    want, _ = O.parallel_solve(A, p, f)
    x, st = _solve(cuda, A, p, f)
    assert st.speculative == 1
    assert st.certificate <= 1e-14
    assert O.rel_err(x, want) <= 1e-12
    assert O.residual(A, x, f) <= 1e-13


@pytest.mark.parametrize("m", [2, 4])
@pytest.mark.parametrize("offs", [(1, 0), (0, 1), (3, 2)])
def test_blktri_unaligned_buffers(cuda, m, offs):
    """A and f 8-byte but not 32-byte aligned: the kernels' scalar loads."""
    NB, p = 40, 5
    n = m * (p * (NB + 1) - 1)
    A = O.generate_random(1, n, m, 1, 1, 60 + m, 4.0)
    f = O.random_vector(n, 4)
    want, _ = O.parallel_solve(A, p, f)
    x, st = _solve(cuda, A, p, f, data_offset=offs[0], f_offset=offs[1])
    assert st.speculative == 1
    assert O.rel_err(x, want) <= 1e-12
