"""TEST INFRASTRUCTURE ONLY -- ctypes front-end for the CPU checkers.

* ``liboracle.so``: the plain-C restatement of the reference hot path
  (oracle/parsol_oracle.c).
* ``_ref/libparsol_ref.so``: the unmodified reference (proj/src) compiled as
  namespace ``parsol_ref`` plus an extern "C" bridge (oracle/ref_bridge.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product (paper_0912_3678_b200) never calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(HERE, "liboracle.so")
_REF_SO = os.path.join(HERE, "_ref", "libparsol_ref.so")

BANDED, BLOCKTRI, ABD, BABD = 0, 1, 2, 3
LU, LUD = 0, 1

_dp = C.POINTER(C.c_double)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"errc {code - 1}: {msg}")
        self.errc = code - 1


class _OrMat(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n", C.c_int), ("m", C.c_int), ("s", C.c_int), ("r", C.c_int),
        ("data", _dp), ("data_len", C.c_size_t), ("corner", _dp),
        ("corner_rows", C.c_int), ("corner_cols", C.c_int), ("abd_off", C.c_void_p),
    ]


def build(ref: bool = True) -> None:
    """Compile the checkers (ref only when /root/reference is present)."""
    targets = ["all"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE_SO):
            build(ref=False)
        L = C.CDLL(_ORACLE_SO)
        L.or_mat_prepare.argtypes = [C.POINTER(_OrMat), C.c_char_p, C.c_size_t]
        L.or_mat_release.argtypes = [C.POINTER(_OrMat)]
        L.or_parallel_factor.argtypes = [C.POINTER(_OrMat), C.c_int, C.c_int,
                                         C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.or_fact_release.argtypes = [C.c_void_p]
        L.or_fact_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 3
        L.or_fact_T.argtypes = [C.c_void_p, _dp]
        L.or_fact_local.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    _dp, _dp, _dp, _dp]
        L.or_solve.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(C.c_longlong), C.c_char_p, C.c_size_t]
        L.or_solve_sequential.argtypes = [C.POINTER(_OrMat), _dp, _dp, C.c_char_p, C.c_size_t]
        L.or_matvec.argtypes = [C.POINTER(_OrMat), _dp, _dp]
        L.or_residual.argtypes = [C.POINTER(_OrMat), _dp, _dp]
        L.or_residual.restype = C.c_double
        L.or_splitmix_unit.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_splitmix_unit.restype = C.c_double
        L.or_config_shape.argtypes = [C.c_int, C.c_int] + [C.POINTER(C.c_int)] * 5 + \
            [C.POINTER(C.c_size_t), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.or_generate_config.argtypes = [C.c_int, C.c_int, C.c_uint64, _dp, _dp, _dp]
        L.or_generate_random.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_double, _dp, _dp]
        L.or_body_entry_count.argtypes = [C.c_int] * 5
        L.or_body_entry_count.restype = C.c_size_t
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            raise FileNotFoundError(_REF_SO + " (build with `make -C oracle ref` where "
                                    "/root/reference is mounted)")
        R = C.CDLL(_REF_SO)
        R.ref_mat_create.argtypes = [C.c_int] * 5 + [_dp, C.c_size_t, _dp, C.c_int, C.c_int]
        R.ref_mat_create.restype = C.c_void_p
        R.ref_mat_destroy.argtypes = [C.c_void_p]
        R.ref_set_threads.argtypes = [C.c_int]
        R.ref_factor.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p), _dp,
                                 C.c_char_p, C.c_size_t]
        R.ref_fact_destroy.argtypes = [C.c_void_p]
        R.ref_factor_tol.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_void_p), C.c_char_p,
                                     C.c_size_t]
        R.ref_fact_layout.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        R.ref_fact_dims.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        R.ref_fact_T.argtypes = [C.c_void_p, _dp]
        R.ref_fact_local.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp]
        R.ref_solve.argtypes = [C.c_void_p, _dp, _dp, C.c_size_t, _dp, C.POINTER(C.c_longlong),
                                C.c_char_p, C.c_size_t]
        R.ref_solve_sequential.argtypes = [C.c_void_p, _dp, _dp, C.c_size_t, C.c_char_p, C.c_size_t]
        R.ref_residual.argtypes = [C.c_void_p, _dp, _dp, C.c_size_t]
        R.ref_residual.restype = C.c_double
        R.ref_plan.argtypes = [C.c_void_p, C.c_int] + [C.POINTER(C.c_int)] * 5 + [C.c_char_p, C.c_size_t]
        R.ref_generate_random.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_double, _dp, _dp, C.c_char_p,
                                                          C.c_size_t]
        vp = C.c_void_p
        R.ref_block_extract.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]
        R.ref_block_extract.restype = vp
        R.ref_block_create.argtypes = [C.c_int] * 9 + [vp] * 6
        R.ref_block_create.restype = vp
        R.ref_block_arrays.argtypes = [vp] * 7
        R.ref_block_destroy.argtypes = [vp]
        R.ref_local_factor.argtypes = [vp, C.c_int, C.c_double, C.POINTER(vp), C.c_char_p, C.c_size_t]
        R.ref_local_destroy.argtypes = [vp]
        R.ref_local_dims.argtypes = [vp, C.POINTER(C.c_int)]
        R.ref_local_field.argtypes = [vp, C.c_int, vp]
        R.ref_local_field.restype = C.c_long
        R.ref_local_op.argtypes = [vp, C.c_int, vp, vp, vp, vp, C.c_char_p, C.c_size_t]
        R.ref_local_dense.argtypes = [vp, C.c_int, vp]
        R.ref_solve_reduced_dense.argtypes = [C.c_int, vp, vp, vp, C.POINTER(C.c_longlong), C.c_char_p,
                                              C.c_size_t]
        _ref = R
    return _ref


@dataclass
class Matrix:
    """A structured matrix in the reference storage layout (structmat.hpp:16-31)."""
    kind: int
    n: int
    m: int
    s: int
    r: int
    data: np.ndarray
    corner: np.ndarray | None = None
    corner_rows: int = 0
    corner_cols: int = 0
    _c: _OrMat | None = field(default=None, repr=False)

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data, dtype=np.float64)
        if self.corner is not None:
            self.corner = np.ascontiguousarray(self.corner, dtype=np.float64)

    def c(self):
        if self._c is None:
            cm = _OrMat(self.kind, self.n, self.m, self.s, self.r, _ptr(self.data), self.data.size,
                        _ptr(self.corner), self.corner_rows, self.corner_cols, None)
            err = C.create_string_buffer(256)
            rc = lib().or_mat_prepare(C.byref(cm), err, 256)
            if rc:
                raise OracleError(rc, err.value.decode())
            self._c = cm
        return C.byref(self._c)

    def __del__(self):
        if self._c is not None and _lib is not None:
            _lib.or_mat_release(C.byref(self._c))


def config_shape(cfg: int, size: int):
    k, n, m, s, r, cr, cc = (C.c_int() for _ in range(7))
    ln = C.c_size_t()
    rc = lib().or_config_shape(cfg, size, C.byref(k), C.byref(n), C.byref(m), C.byref(s), C.byref(r),
                               C.byref(ln), C.byref(cr), C.byref(cc))
    if rc:
        raise OracleError(rc, "bad config")
    return dict(kind=k.value, n=n.value, m=m.value, s=s.value, r=r.value, data_len=ln.value,
                corner_rows=cr.value, corner_cols=cc.value)


def generate_config(cfg: int, size: int, seed: int):
    """Seeded BASELINE config instance -> (Matrix, f)."""
    sh = config_shape(cfg, size)
    data = np.empty(sh["data_len"], np.float64)
    corner = np.empty(64, np.float64) if cfg == 4 else None
    f = np.empty(sh["n"], np.float64)
    lib().or_generate_config(cfg, size, seed, _ptr(data), _ptr(corner), _ptr(f))
    A = Matrix(sh["kind"], sh["n"], sh["m"], sh["s"], sh["r"], data, corner,
               sh["corner_rows"], sh["corner_cols"])
    return A, f


def generate_random(kind: int, n: int, m: int, s: int, r: int, seed: int, dominance: float):
    """Restated generate_random (src/structmat.cpp:282-333) -> Matrix."""
    cnt = lib().or_body_entry_count(kind, n, m, s, r)
    data = np.empty(cnt, np.float64)
    corner = np.empty(m * m, np.float64) if kind == BABD else None
    rc = lib().or_generate_random(kind, n, m, s, r, seed, dominance, _ptr(data), _ptr(corner))
    if rc:
        raise OracleError(rc, "generate_random failed")
    return Matrix(kind, n, m, s, r, data, corner, m if kind == BABD else 0, m if kind == BABD else 0)


def random_vector(n: int, seed: int):
    """tests/oracles.hpp:42-47: SplitMix64(seed, 77) draws."""
    return np.array([lib().or_splitmix_unit(seed, 77, k + 1) for k in range(n)])


def parallel_solve(A: Matrix, p: int, f: np.ndarray, strategy: int = LU):
    """Restated parallel_factor + solve -> (x, reduced_ops)."""
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib().or_parallel_factor(A.c(), p, strategy, C.byref(h), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    try:
        f = np.ascontiguousarray(f, np.float64)
        x = np.empty(A.n, np.float64)
        ops = C.c_longlong(0)
        rc = lib().or_solve(h, _ptr(f), _ptr(x), C.byref(ops), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return x, ops.value
    finally:
        lib().or_fact_release(h)


def factor_info(A: Matrix, p: int, strategy: int = LU, want_T: bool = True):
    """Restated parallel_factor -> dict(q, dim, k, T (dense or None), locals list)."""
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib().or_parallel_factor(A.c(), p, strategy, C.byref(h), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    try:
        q, dim, k = C.c_int(), C.c_int(), C.c_int()
        lib().or_fact_dims(h, C.byref(q), C.byref(dim), C.byref(k))
        T = None
        if want_T:
            T = np.empty((dim.value, dim.value), np.float64)
            lib().or_fact_T(h, _ptr(T))
        locs = []
        kk = k.value
        for i in range(p):
            k0, k1 = C.c_int(), C.c_int()
            a1, a2, b, g = (np.zeros(kk * kk) for _ in range(4))
            lib().or_fact_local(h, i, C.byref(k0), C.byref(k1), _ptr(a1), _ptr(a2), _ptr(b), _ptr(g))
            locs.append(dict(k0=k0.value, k1=k1.value,
                             alpha1=a1[:k0.value ** 2].reshape(k0.value, k0.value),
                             alpha2=a2[:k1.value ** 2].reshape(k1.value, k1.value),
                             beta=b[:k1.value * k0.value].reshape(k1.value, k0.value),
                             gamma=g[:k0.value * k1.value].reshape(k0.value, k1.value)))
        return dict(q=q.value, dim=dim.value, k=kk, T=T, locals=locs)
    finally:
        lib().or_fact_release(h)


def solve_sequential(A: Matrix, f: np.ndarray):
    f = np.ascontiguousarray(f, np.float64)
    x = np.empty(A.n, np.float64)
    err = C.create_string_buffer(512)
    rc = lib().or_solve_sequential(A.c(), _ptr(f), _ptr(x), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return x


def matvec(A: Matrix, x: np.ndarray):
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(A.n, np.float64)
    lib().or_matvec(A.c(), _ptr(x), _ptr(y))
    return y


def residual(A: Matrix, x: np.ndarray, f: np.ndarray) -> float:
    x = np.ascontiguousarray(x, np.float64)
    f = np.ascontiguousarray(f, np.float64)
    return lib().or_residual(A.c(), _ptr(x), _ptr(f))


def rel_err(got, want) -> float:
    """Normwise infinity relative error (tests/oracles.hpp:61-68)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    num = float(np.max(np.abs(got - want))) if got.size else 0.0
    den = float(np.max(np.abs(want))) if want.size else 0.0
    return num / den if den > 0 else num


# --------------------------------------------------------------------------
# The unmodified reference (oracle/_ref)
# --------------------------------------------------------------------------

class RefMatrix:
    def __init__(self, A: Matrix):
        self.n = A.n
        self._keep = A
        self.h = ref().ref_mat_create(A.kind, A.n, A.m, A.s, A.r, _ptr(A.data), A.data.size,
                                      _ptr(A.corner), A.corner_rows, A.corner_cols)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_mat_destroy(self.h)
            self.h = None

    def factor(self, p: int, strategy: int = LU):
        h = C.c_void_p()
        secs = C.c_double()
        err = C.create_string_buffer(512)
        rc = ref().ref_factor(self.h, p, strategy, C.byref(h), C.byref(secs), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return RefFact(h, self.n, secs.value)

    def factor_tol(self, p: int, strategy: int, tol: float):
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = ref().ref_factor_tol(self.h, p, strategy, tol, C.byref(h), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return RefFact(h, self.n, 0.0)

    def solve_sequential(self, f):
        f = np.ascontiguousarray(f, np.float64)
        x = np.empty(self.n, np.float64)
        err = C.create_string_buffer(512)
        rc = ref().ref_solve_sequential(self.h, _ptr(f), _ptr(x), self.n, err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return x

    def residual(self, x, f) -> float:
        x = np.ascontiguousarray(x, np.float64)
        f = np.ascontiguousarray(f, np.float64)
        return ref().ref_residual(self.h, _ptr(x), _ptr(f), self.n)

    def plan(self, p: int):
        bb = (C.c_int * p)()
        be = (C.c_int * p)()
        ss = (C.c_int * (p + 1))()
        cnt, k = C.c_int(), C.c_int()
        err = C.create_string_buffer(512)
        rc = ref().ref_plan(self.h, p, bb, be, ss, C.byref(cnt), C.byref(k), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return dict(body=[(bb[i], be[i]) for i in range(p)], seps=list(ss[:cnt.value]), k=k.value)


class RefFact:
    def __init__(self, h, n, secs):
        self.h, self.n, self.factor_seconds = h, n, secs

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_fact_destroy(self.h)
            self.h = None

    def dims(self):
        q, dim = C.c_int(), C.c_int()
        ref().ref_fact_dims(self.h, C.byref(q), C.byref(dim))
        return q.value, dim.value

    def layout(self):
        q, _ = self.dims()
        pos = np.empty(q, np.int32)
        size = np.empty(q, np.int32)
        ref().ref_fact_layout(self.h, pos.ctypes.data, size.ctypes.data)
        return pos, size

    def T(self):
        _, dim = self.dims()
        T = np.empty((dim, dim), np.float64)
        ref().ref_fact_T(self.h, _ptr(T))
        return T

    def solve(self, f):
        f = np.ascontiguousarray(f, np.float64)
        x = np.empty(self.n, np.float64)
        ph = np.zeros(3)
        ops = C.c_longlong()
        err = C.create_string_buffer(512)
        rc = ref().ref_solve(self.h, _ptr(f), _ptr(x), self.n, _ptr(ph), C.byref(ops), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return x, ops.value, ph


def ref_generate_random(kind, n, m, s, r, seed, dominance):
    cnt = lib().or_body_entry_count(kind, n, m, s, r)
    data = np.empty(cnt, np.float64)
    corner = np.empty(m * m, np.float64) if kind == BABD else None
    err = C.create_string_buffer(256)
    rc = ref().ref_generate_random(kind, n, m, s, r, seed, dominance, _ptr(data), _ptr(corner), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    return data, corner


def ref_set_threads(t: int) -> int:
    return ref().ref_set_threads(t)


# --------------------------------------------------------------------------
# The reference's per-partition API (extract_block, factor, LocalFactorization
# members) -- the parity target of psg_local_* (tests/test_localfact_gpu.py)
# --------------------------------------------------------------------------

def ref_extract_block(A, p: int, i: int) -> dict:
    """extract_block(A, plan_partition(A, p), i) of the reference, as arrays
    (A: a Matrix, or a RefMatrix to reuse its reference copy)."""
    R = A if isinstance(A, RefMatrix) else RefMatrix(A)
    A = R._keep
    dims = (C.c_int * 5)()
    err = C.create_string_buffer(512)
    hb = ref().ref_block_extract(R.h, p, i, dims, err, 512)
    if not hb:
        raise OracleError(1, err.value.decode())
    L, k0, k1, es, er = list(dims)
    out = dict(kind=A.kind, m=A.m, s=A.s, r=A.r, L=L, k0=k0, k1=k1, env_s=es, env_r=er,
               env=np.zeros(L * (es + 1 + er)), b0=np.zeros(L * k0), c0=np.zeros(L * k0), b1=np.zeros(L * k1),
               c1=np.zeros(L * k1), a_right=np.zeros(k1 * k1))
    ref().ref_block_arrays(hb, *(out[k].ctypes.data for k in ("env", "b0", "c0", "b1", "c1", "a_right")))
    ref().ref_block_destroy(hb)
    return out


class RefLocal:
    """The reference's LocalFactorization of one block (factor(strategy, blk, tol))."""

    def __init__(self, blk: dict, strategy: int, tol: float = 1e-8):
        arr = {k: np.ascontiguousarray(blk[k], np.float64) for k in ("env", "b0", "c0", "b1", "c1", "a_right")}
        self._keep = arr
        hb = ref().ref_block_create(blk["kind"], blk["m"], blk["s"], blk["r"], blk["L"], blk["k0"], blk["k1"],
                                    blk["env_s"], blk["env_r"],
                                    *(arr[k].ctypes.data if arr[k].size else None
                                      for k in ("env", "b0", "c0", "b1", "c1", "a_right")))
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = ref().ref_local_factor(hb, strategy, tol, C.byref(h), err, 512)
        ref().ref_block_destroy(hb)
        if rc:
            raise OracleError(rc, err.value.decode())
        self.h = h
        d = (C.c_int * 9)()
        ref().ref_local_dims(h, d)
        self.kept_dim, self.n_extras, self.cr_levels, self.core, self.dim, self.n_a_order, self.n_elims, self.g, \
            self.n_rem = list(d)
        self.L = blk["L"]

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_local_destroy(self.h)
            self.h = None

    def field(self, fid: int, count: int, dtype=np.float64):
        out = np.zeros(max(count, 1), dtype)
        n = ref().ref_local_field(self.h, fid, out.ctypes.data)
        return out[:n]

    def op(self, op: int, v, v2=None):
        v = np.ascontiguousarray(v, np.float64)
        v2 = None if v2 is None else np.ascontiguousarray(v2, np.float64)
        out = np.empty(self.L)
        out2 = np.empty(max(self.kept_dim, 1))
        err = C.create_string_buffer(512)
        rc = ref().ref_local_op(self.h, op, v.ctypes.data, None if v2 is None else v2.ctypes.data, out.ctypes.data,
                                out2.ctypes.data, err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return (out, out2[:self.kept_dim]) if op == 0 else out

    def dense(self, which: int):
        M = np.empty((self.dim, self.dim))
        ref().ref_local_dense(self.h, which, M.ctypes.data)
        return M


def ref_solve_reduced_dense(T, rhs):
    T = np.ascontiguousarray(T, np.float64)
    rhs = np.ascontiguousarray(rhs, np.float64)
    x = np.empty(rhs.size)
    ops = C.c_longlong()
    err = C.create_string_buffer(512)
    rc = ref().ref_solve_reduced_dense(rhs.size, T.ctypes.data, rhs.ctypes.data, x.ctypes.data, C.byref(ops), err,
                                       512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return x, ops.value
