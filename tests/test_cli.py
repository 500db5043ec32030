"""The `psg` command-line tool (paper_0912_3678_b200/cli/psg.cpp) and its
STRUCTMAT / VEC files (include/parsol/io.hpp).

CPU: files written by `psg generate` are byte-identical to the reference
writer's (src/io.cpp, compiled unmodified into oracle/_ref) for the same
matrix and comment, and parse back through the reference parser to the same
data; plan output; usage / parse / I/O errors and exit codes.
GPU: solve / verify / bench, exit code 2 on a numeric failure (SPEC.md
"MODULE cli")."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PSG = os.path.join(ROOT, "paper_0912_3678_b200", "psg")


@pytest.fixture(scope="module")
def psg_bin():
    from paper_0912_3678_b200 import build
    build.build(verbose=False)
    return PSG


def run(*args, cwd=None):
    return subprocess.run([PSG, *map(str, args)], capture_output=True, text=True, cwd=cwd)


def _ref_lib():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    lib = O.ref()
    lib.ref_write_matrix.restype = C.c_long
    lib.ref_write_matrix.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_size_t]
    lib.ref_write_vector.restype = C.c_long
    lib.ref_write_vector.argtypes = [C.c_void_p, C.c_size_t, C.c_char_p, C.c_char_p, C.c_size_t]
    lib.ref_parse_matrix.restype = C.c_int
    lib.ref_parse_matrix.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    lib.ref_mat_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 5 + [C.POINTER(C.c_size_t), C.c_void_p]
    return lib


@pytest.mark.parametrize("kind,name,n,m,s,r", [(0, "banded", 300, 1, 2, 1), (1, "blocktri", 96, 4, 1, 1),
                                               (2, "abd", 120, 4, 2, 2), (3, "babd", 64, 4, 2, 2)])
def test_generate_matches_reference_writer(psg_bin, tmp_path, kind, name, n, m, s, r):
    lib = _ref_lib()
    out = tmp_path / "a.mat"
    res = run("generate", "--kind", name, "--n", n, "--m", m, "--s", s, "--r", r, "--seed", 5, "--dominance", 2,
              "-o", out)
    assert res.returncode == 0, res.stderr
    ours = out.read_bytes()
    # the same matrix through the reference generator and writer
    A = O.RefMatrix(O.generate_random(kind, n, m, s, r, 5, 2.0))
    comment = b"generator generate_random splitmix64 seed 5 dominance 0x1p+1"
    cap = len(ours) + 4096
    buf = C.create_string_buffer(cap)
    ln = lib.ref_write_matrix(A.h, comment, buf, cap)
    assert buf.raw[:ln] == ours
    # and back through the reference parser
    h = C.c_void_p()
    err = C.create_string_buffer(256)
    assert lib.ref_parse_matrix(ours, len(ours), C.byref(h), err, 256) == 0, err.value
    k, nn, mm, ss, rr = (C.c_int() for _ in range(5))
    ln2 = C.c_size_t()
    lib.ref_mat_dims(h, C.byref(k), C.byref(nn), C.byref(mm), C.byref(ss), C.byref(rr), C.byref(ln2), None)
    data = np.empty(ln2.value)
    lib.ref_mat_dims(h, C.byref(k), C.byref(nn), C.byref(mm), C.byref(ss), C.byref(rr), C.byref(ln2),
                     data.ctypes.data_as(C.c_void_p))
    lib.ref_mat_destroy(h)
    assert (k.value, nn.value, mm.value, ss.value, rr.value) == (kind, n, m, s, r)
    assert np.array_equal(data, O.generate_random(kind, n, m, s, r, 5, 2.0).data)


def test_rhs_vector_matches_reference_writer(psg_bin, tmp_path):
    lib = _ref_lib()
    res = run("generate", "--kind", "banded", "--n", 50, "--seed", 2, "-o", tmp_path / "a.mat", "--rhs",
              tmp_path / "f.vec")
    assert res.returncode == 0, res.stderr
    ours = (tmp_path / "f.vec").read_bytes()
    v = np.ones(50)
    buf = C.create_string_buffer(len(ours) + 1024)
    ln = lib.ref_write_vector(v.ctypes.data_as(C.c_void_p), 50,
                              b"generator generate_random splitmix64 seed 2 dominance 0x1p+1", buf, len(ours) + 1024)
    assert buf.raw[:ln] == ours


def test_plan_and_errors(psg_bin, tmp_path):
    res = run("generate", "--kind", "banded", "--n", 100, "--seed", 1, "-o", tmp_path / "a.mat")
    assert res.returncode == 0
    res = run("plan", "-m", tmp_path / "a.mat", "--p", 4)
    assert res.returncode == 0 and "A(1) rows [0, 25)" in res.stdout and "a(3) at 75" in res.stdout
    res = run("plan", "-m", tmp_path / "missing.mat", "--p", 4)
    assert res.returncode == 1 and res.stderr.startswith("ERROR IoError")
    (tmp_path / "bad.mat").write_text("STRUCTMAT 2 banded 3 1 1 1\n")
    res = run("plan", "-m", tmp_path / "bad.mat", "--p", 2)
    assert res.returncode == 1 and res.stderr.startswith("ERROR UnsupportedVersion")
    res = run("plan", "-m", tmp_path / "a.mat", "--p", 1)
    assert res.returncode == 1 and res.stderr.startswith("ERROR TooManyPartitions")
    res = run("frobnicate")
    assert res.returncode == 1 and res.stderr.startswith("ERROR InvalidParameter")


@pytest.mark.gpu
def test_solve_and_verify(psg_bin, tmp_path, cuda):
    """SPEC cli examples: generate + solve -> residual <= 1e-10 printed; verify -> exit 0."""
    res = run("generate", "--kind", "banded", "--n", 100, "--s", 1, "--r", 1, "--seed", 1, "--dominance", 2,
              "-o", tmp_path / "a.mat")
    assert res.returncode == 0
    res = run("solve", "-m", tmp_path / "a.mat", "-f", "ones", "--p", 4, "--strategy", "lu", "-o", tmp_path / "x.vec")
    assert res.returncode == 0, res.stderr
    resid = float(res.stdout.split()[2].strip("()"))
    assert resid <= 1e-10
    x = np.array([float.fromhex(t) for t in (tmp_path / "x.vec").read_text().split("\n")[1:] if t])
    A = O.generate_random(0, 100, 1, 1, 1, 1, 2.0)
    assert O.rel_err(x, O.solve_sequential(A, np.ones(100))) <= 1e-12
    for kind, extra in (("blocktri", ["--m", 4]), ("babd", ["--m", 4, "--s", 2, "--r", 2])):
        run("generate", "--kind", kind, "--n", 96, *extra, "--seed", 3, "-o", tmp_path / "b.mat")
        res = run("verify", "-m", tmp_path / "b.mat", "-f", "ones", "--p", 3)
        assert res.returncode == 0, res.stdout + res.stderr
        assert "max relative error" in res.stdout


@pytest.mark.gpu
def test_config_generate_and_bench(psg_bin, tmp_path, cuda):
    res = run("generate", "--config", 4, "--size", 255, "--seed", 3, "-o", tmp_path / "c4.mat", "--rhs",
              tmp_path / "c4.vec")
    assert res.returncode == 0, res.stderr
    want_A, want_f = O.generate_config(4, 255, 3)
    lines = [t for t in (tmp_path / "c4.mat").read_text().split("\n")[1:] if t and not t.startswith("#")]
    vals = np.array([float.fromhex(t) for t in lines])
    assert np.array_equal(vals[:want_A.data.size], want_A.data)  # device generator == CPU restatement, bit-exact
    assert np.array_equal(vals[want_A.data.size:], want_A.corner)
    res = run("verify", "-m", tmp_path / "c4.mat", "-f", tmp_path / "c4.vec", "--p", 8)
    assert res.returncode == 0, res.stdout + res.stderr
    res = run("bench", "--config", 1, "--size", 1 << 16, "--p", 64, "--reps", 3)
    assert res.returncode == 0, res.stderr
    rows = res.stdout.strip().split("\n")
    assert rows[0] == "phase,n,p,workers,median_seconds,op_count"
    assert [r.split(",")[0] for r in rows[1:]] == ["factor", "phase1", "phase2", "phase3", "total"]


@pytest.mark.gpu
def test_numeric_failure_exit_code(psg_bin, tmp_path, cuda):
    """A zero pivot in a body -> exit 2 and a machine-readable error line."""
    n = 40
    sub, diag, sup = np.zeros(n - 1), np.ones(n), np.zeros(n - 1)
    diag[5] = 0.0
    body = np.concatenate([sub, diag, sup])
    txt = "STRUCTMAT 1 banded %d 1 1 1\n" % n + "".join(float.hex(float(v)) + "\n" for v in body)
    (tmp_path / "z.mat").write_text(txt)
    res = run("solve", "-m", tmp_path / "z.mat", "-f", "ones", "--p", 2)
    assert res.returncode == 2, res.stdout + res.stderr
    assert res.stderr.startswith("ERROR ")


def _traj(path):
    lines = [t for t in path.read_text().split("\n") if t and not t.startswith("#")]
    head = lines[0].split()
    assert head[:2] == ["TRAJ", "1"]
    m, p, N = (int(v) for v in head[2:5])
    vals = np.array([float.fromhex(t) for t in lines[1:]])
    return vals.reshape(p * N + 1, m)


@pytest.mark.gpu
def test_ode_and_parareal_commands(psg_bin, tmp_path, cuda):
    """`ode` writes a TRAJ file equal to the reference's trajectory; `parareal`
    prints the `iter,update_norm` CSV of the reference's iteration, exit 2 on
    non-convergence (SPEC cli)."""
    import ctypes as C
    m, p, N = 8, 4, 25
    res = run("ode", "--problem", "heat", "--m", m, "--p", p, "--N", N, "--method", "trap", "-o", tmp_path / "y.traj")
    assert res.returncode == 0, res.stderr
    Y = _traj(tmp_path / "y.traj")
    inv = float(m + 1) ** 2
    L = np.ascontiguousarray(np.diag(-2 * inv * np.ones(m)) + np.diag(inv * np.ones(m - 1), 1) +
                             np.diag(inv * np.ones(m - 1), -1))
    y0 = np.sin(np.pi * np.arange(1, m + 1) / (m + 1))
    want = np.zeros((p * N + 1) * m)
    err = C.create_string_buffer(256)
    G = C.CFUNCTYPE(None, C.c_double, C.POINTER(C.c_double), C.c_void_p)
    rc = O.ref().ref_ode_solve(C.c_int(m), L.ctypes.data_as(C.c_void_p), y0.ctypes.data_as(C.c_void_p),
                               C.c_double(0.0), C.c_double(0.1), C.c_int(p), C.c_int(N), C.c_int(1),
                               C.cast(None, G), C.c_void_p(None), C.c_int(0), want.ctypes.data_as(C.c_void_p), err,
                               C.c_size_t(256))
    assert rc == 0, err.value
    assert O.rel_err(Y.ravel(), want) <= 1e-12
    res = run("parareal", "--problem", "heat", "--m", 16, "--p", 8, "--N", 50, "-o", tmp_path / "h.csv")
    assert res.returncode == 0, res.stderr
    rows = (tmp_path / "h.csv").read_text().strip().split("\n")
    assert rows[0] == "iter,update_norm" and len(rows) > 2
    it = int(res.stdout.split()[1])
    assert it == len(rows) - 1
    res = run("parareal", "--problem", "heat", "--m", 16, "--p", 8, "--N", 50, "--tol", "1e-15", "--max-iter", 1)
    assert res.returncode == 2 and res.stderr.startswith("ERROR NotConverged")


@pytest.mark.gpu
def test_pivoting_strategy_command(psg_bin, tmp_path, cuda):
    res = run("generate", "--kind", "circulant", "--n", 200, "--s", 1, "--r", 1, "--seed", 5, "--dominance", 1,
              "-o", tmp_path / "c.mat")
    assert res.returncode == 0, res.stderr
    for st in ("lupivot", "qr"):
        res = run("verify", "-m", tmp_path / "c.mat", "-f", "ones", "--p", 4, "--strategy", st)
        assert res.returncode == 0, res.stdout + res.stderr


@pytest.mark.parametrize("kind,name,n,m,s,r", [(0, "banded", 300, 1, 2, 1), (0, "banded", 40, 1, 3, 3),
                                               (1, "blocktri", 96, 4, 1, 1), (2, "abd", 120, 4, 2, 2),
                                               (3, "babd", 64, 4, 2, 2), (4, "circulant", 50, 1, 2, 1),
                                               (4, "circulant", 7, 1, 3, 3)])
def test_generate_random_matches_unmodified_reference(psg_bin, tmp_path, kind, name, n, m, s, r):
    """generate_random of this library (the dominance pass walks each row's
    stored columns: O(nnz)) against the UNMODIFIED reference's generator, every
    kind incl. circulant-like (its diagonal lives in band s) and tiny n where
    a circulant row lists a column twice."""
    _ref_lib()
    out = tmp_path / "g.mat"
    res = run("generate", "--kind", name, "--n", n, "--m", m, "--s", s, "--r", r, "--seed", 9, "--dominance", 2,
              "-o", out)
    assert res.returncode == 0, res.stderr
    lib = O.ref()
    lib.ref_parse_matrix.restype = C.c_int
    lib.ref_parse_matrix.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    lib.ref_mat_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 5 + [C.POINTER(C.c_size_t), C.c_void_p]
    text = out.read_bytes()
    h = C.c_void_p()
    err = C.create_string_buffer(256)
    assert lib.ref_parse_matrix(text, len(text), C.byref(h), err, 256) == 0, err.value
    k, nn, mm, ss, rr = (C.c_int() for _ in range(5))
    ln = C.c_size_t()
    lib.ref_mat_dims(h, C.byref(k), C.byref(nn), C.byref(mm), C.byref(ss), C.byref(rr), C.byref(ln), None)
    ours = np.empty(ln.value)
    lib.ref_mat_dims(h, C.byref(k), C.byref(nn), C.byref(mm), C.byref(ss), C.byref(rr), C.byref(ln),
                     ours.ctypes.data_as(C.c_void_p))
    lib.ref_mat_destroy(h)
    want, _ = O.ref_generate_random(kind, n, m, s, r, 9, 2.0)
    assert np.array_equal(ours, want)


def test_generate_is_linear_time(psg_bin, tmp_path):
    """psg generate of a 2^24-row dominant banded matrix finishes in seconds
    (generate_random walks each row's structure, not all n columns)."""
    import time
    t0 = time.perf_counter()
    res = run("generate", "--kind", "banded", "--n", 1 << 24, "--s", 1, "--r", 1, "--seed", 1, "--dominance", 2,
              "-o", "/dev/null")
    dt = time.perf_counter() - t0
    assert res.returncode == 0, res.stderr
    assert dt < 60, dt
