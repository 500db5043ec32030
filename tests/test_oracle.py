"""CPU checks of the oracle (test infrastructure): the plain-C restatement is
pinned bit-for-bit to the committed golden fixtures produced by the unmodified
reference (tests/golden/make_golden.py), to the SPEC.md known answers, and --
when oracle/_ref is built -- to the live reference on fresh random cases."""
import glob
import hashlib
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = sorted(glob.glob(os.path.join(GOLD, "cfg*.npz")))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(c)[:-4] for c in CASES])
def test_oracle_matches_reference_golden(path):
    g = np.load(path)
    A, f = O.generate_config(int(g["cfg"]), int(g["size"]), int(g["seed"]))
    assert _sha(A.data) == str(g["data_sha"]) and _sha(f) == str(g["f_sha"]), "generator drifted"
    x, ops = O.parallel_solve(A, int(g["p"]), f)
    assert np.array_equal(x, g["x"]), "parallel_factor+solve restatement is not bit-identical"
    assert ops == int(g["reduced_ops"])
    assert np.array_equal(O.solve_sequential(A, f), g["x_seq"])
    assert O.residual(A, x, f) == float(g["residual"])
    info = O.factor_info(A, int(g["p"]), want_T=g["T"].size > 0)
    assert info["q"] == int(g["q"]) and info["dim"] == int(g["dim"])
    if g["T"].size:
        assert np.array_equal(info["T"], g["T"])


def test_known_answers():
    kat = np.load(os.path.join(GOLD, "kat.npz"))
    T3 = O.Matrix(O.BANDED, 3, 1, 1, 1, np.array([-1.0, -1.0, 2.0, 2.0, 2.0, -1.0, -1.0]))
    x, _ = O.parallel_solve(T3, 2, np.ones(3))
    assert np.allclose(x, [1.5, 2.0, 1.5], rtol=0, atol=1e-15)
    assert np.array_equal(x, kat["toeplitz3_x"])
    T9 = O.Matrix(O.BANDED, 9, 1, 1, 1, np.concatenate([-np.ones(8), 2 * np.ones(9), -np.ones(8)]))
    assert O.factor_info(T9, 2)["q"] == 1 == int(kat["toeplitz9_q"])
    I8 = O.Matrix(O.BANDED, 8, 1, 1, 1, np.concatenate([np.zeros(7), np.ones(8), np.zeros(7)]))
    x, _ = O.parallel_solve(I8, 4, np.arange(1.0, 9.0))
    assert np.array_equal(x, np.arange(1.0, 9.0))                          # identity -> x = f
    info = O.factor_info(I8, 4)
    assert np.array_equal(info["T"], np.eye(3))                            # SPEC.md:304 T_p = I


def test_oracle_errors():
    A, f = O.generate_config(0, 100, 1)
    with pytest.raises(O.OracleError) as e:
        O.parallel_solve(A, 1, f)
    assert e.value.errc == 7  # TooManyPartitions
    with pytest.raises(O.OracleError) as e:
        O.parallel_solve(A, 60, f)
    assert e.value.errc == 7
    bad = O.Matrix(O.BANDED, 100, 1, 1, 1, A.data[:-1])
    with pytest.raises(O.OracleError) as e:
        bad.c()
    assert e.value.errc == 0  # DimensionMismatch


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("cfg,size,p,strategy", [(0, 3000, 7, O.LU), (0, 3000, 7, O.LUD), (2, 100, 5, O.LU),
                                                 (3, 2000, 9, O.LUD), (4, 200, 6, O.LU), (4, 64, 4, O.LUD)])
def test_restatement_vs_live_reference(cfg, size, p, strategy):
    A, f = O.generate_config(cfg, size, 1234 + size)
    x, ops = O.parallel_solve(A, p, f, strategy)
    R = O.RefMatrix(A)
    xr, opsr, _ = R.factor(p, strategy).solve(f)
    assert np.array_equal(x, xr) and ops == opsr
    assert np.array_equal(O.solve_sequential(A, f), R.solve_sequential(f))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_zero_pivot_partition_matches_reference():
    n, p = 3000, 3
    d = np.concatenate([np.ones(n - 1), 4 * np.ones(n), np.ones(n - 1)])
    d[n - 1 + 1001] = 0.0
    d[n - 1 + 1002] = 0.0
    A = O.Matrix(O.BANDED, n, 1, 1, 1, d)
    with pytest.raises(O.OracleError) as eo:
        O.parallel_solve(A, p, np.ones(n))
    with pytest.raises(O.OracleError) as er:
        O.RefMatrix(A).factor(p)
    assert eo.value.errc == er.value.errc == 11
    assert "partition 2" in str(eo.value) and "partition 2" in str(er.value)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("kind,n,m,s,r", [(0, 37, 1, 2, 3), (1, 36, 3, 1, 1), (2, 40, 4, 2, 2), (3, 44, 2, 1, 1)])
def test_generate_random_matches_reference(kind, n, m, s, r):
    A = O.generate_random(kind, n, m, s, r, 17, 2.0)
    d, c = O.ref_generate_random(kind, n, m, s, r, 17, 2.0)
    assert np.array_equal(A.data, d)
    if c is not None:
        assert np.array_equal(A.corner, c)
