"""paper_0912_3678_b200 -- B200-native partition solver (A = F T G, arXiv 0912.3678).

Python mirror of the reference `parsol` solver API (proj/include/parsol/
parfact.hpp:52-63) over the C ABI in include/psg.h (libpsg.so, sm_100a).  The
names, argument meaning and error behaviour follow the reference:

    F = parallel_factor(A, p, Strategy.Lu)      # parsol::parallel_factor
    x = solve(F, f, stats)                      # parsol::solve
    r = residual(A, x, f)                       # parsol::residual

Vectors may be numpy arrays (host; copied through the handle) or CUDA torch
tensors (device-resident; no copies).  There is no CPU fallback: importing the
solver on a machine without the built extension raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Any

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIBPSG = os.path.join(_PKG, "libpsg.so")

__all__ = ["Kind", "Strategy", "Errc", "Error", "StructuredMatrix", "ParallelFactorization",
           "SolveStats", "parallel_factor", "solve", "solve_reduced", "residual", "matvec",
           "plan_partition", "generate_config", "config_shape", "lib", "PartitionBlock", "LocalFactorization",
           "factor", "factor_lu", "factor_lud", "factor_cyclic_reduction", "factor_lu_pivot", "factor_qr",
           "dense_solve"]


class Kind(enum.IntEnum):  # include/parsol/structmat.hpp:11
    Banded = 0
    BlockTridiagonal = 1
    Abd = 2
    Babd = 3
    CirculantLike = 4


class Strategy(enum.IntEnum):  # include/parsol/localfact.hpp:11
    Lu = 0
    Lud = 1
    CyclicReduction = 2
    Arce = 3
    LuPivot = 4
    Qr = 5


class Errc(enum.IntEnum):  # include/parsol/errors.hpp:12-35
    DimensionMismatch = 0
    InvalidBandwidth = 1
    CornerForbidden = 2
    TooLargeForDense = 3
    InvalidParameter = 4
    ParseError = 5
    UnsupportedVersion = 6
    TooManyPartitions = 7
    UnsupportedKind = 8
    UnsupportedStructure = 9
    IndexOutOfRange = 10
    ZeroPivot = 11
    SingularBlock = 12
    SingularFactor = 13
    SingularReducedSystem = 14
    SingularWindow = 15
    ExhaustedBody = 16
    StepTooLarge = 17
    InvalidInterval = 18
    ExpmFailure = 19
    NotConverged = 20
    IoError = 21
    Cuda = 100


class Error(RuntimeError):
    """parsol::Error: carries the reference error code (errors.hpp:39-51)."""

    def __init__(self, code: int, detail: str):
        try:
            c = Errc(code)
            name = c.name
        except ValueError:
            c, name = code, f"Errc{code}"
        super().__init__(f"{name}: {detail}")
        self.code = c
        self.detail = detail


class _Desc(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int), ("m", C.c_int), ("s", C.c_int), ("r", C.c_int),
                ("data", C.c_void_p), ("data_len", C.c_size_t), ("corner", C.c_void_p),
                ("corner_rows", C.c_int), ("corner_cols", C.c_int), ("on_device", C.c_int)]


class _Block(C.Structure):  # psg_block
    _fields_ = [("kind", C.c_int), ("m", C.c_int), ("s", C.c_int), ("r", C.c_int), ("L", C.c_int),
                ("k0", C.c_int), ("k1", C.c_int), ("env_s", C.c_int), ("env_r", C.c_int),
                ("env", C.c_void_p), ("b0", C.c_void_p), ("c0", C.c_void_p), ("b1", C.c_void_p),
                ("c1", C.c_void_p), ("a_right", C.c_void_p)]


class _LocalInfo(C.Structure):  # psg_local_info
    _fields_ = [(k, C.c_int) for k in ("strategy", "L", "k0", "k1", "env_s", "env_r", "core", "cr_levels", "g",
                                        "n_elims", "n_rem")] + \
               [("rem", C.c_int * 2)] + [(k, C.c_int) for k in ("dim", "n_a_order", "n_extras")]


class SolveStats(C.Structure):
    """parsol::SolveStats (parfact.hpp:24-30) + the GPU certificate."""
    _fields_ = [("factor_seconds", C.c_double), ("phase1_seconds", C.c_double),
                ("phase2_seconds", C.c_double), ("phase3_seconds", C.c_double),
                ("reduced_ops", C.c_longlong), ("certificate", C.c_double),
                ("speculative", C.c_int), ("fallbacks", C.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libpsg.so (raises if the CUDA extension is missing -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIBPSG):
            raise ImportError(f"{_LIBPSG} is missing: build it with `python -m paper_0912_3678_b200.build` "
                              "(the GPU path has no CPU fallback)")
        L = C.CDLL(_LIBPSG)
        vp, ip, sz, cp = C.c_void_p, C.c_int, C.c_size_t, C.c_char_p
        L.psg_factor.argtypes = [C.POINTER(_Desc), ip, ip, C.c_double, vp, C.POINTER(vp), cp, sz]
        L.psg_solve.argtypes = [vp, vp, vp, ip, vp, C.POINTER(SolveStats), cp, sz]
        L.psg_solve_async.argtypes = [vp, vp, vp, ip, vp, cp, sz]
        L.psg_sync.argtypes = [vp, C.POINTER(SolveStats), cp, sz]
        L.psg_refactor.argtypes = [vp, C.POINTER(_Desc), vp, cp, sz]
        L.psg_release.argtypes = [vp]
        L.psg_release.restype = None
        L.psg_reduced_info.argtypes = [vp] + [C.POINTER(C.c_int)] * 4
        L.psg_reduced_blocks.argtypes = [vp, vp, vp, vp, cp, sz]
        L.psg_reduced_layout.argtypes = [vp, vp, vp]
        L.psg_reduced_dense.argtypes = [vp, vp, cp, sz]
        L.psg_solve_reduced.argtypes = [vp, vp, vp, ip, vp, C.POINTER(SolveStats), cp, sz]
        L.psg_plan.argtypes = [C.POINTER(_Desc), ip] + [C.POINTER(C.c_int)] * 5 + [cp, sz]
        L.psg_residual.argtypes = [C.POINTER(_Desc), vp, vp, ip, vp, C.POINTER(C.c_double), cp, sz]
        L.psg_matvec.argtypes = [C.POINTER(_Desc), vp, vp, ip, vp, cp, sz]
        L.psg_config_shape.argtypes = [ip, ip] + [C.POINTER(C.c_int)] * 5 + \
            [C.POINTER(C.c_size_t), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.psg_generate_config.argtypes = [ip, ip, C.c_uint64, vp, vp, vp, vp, cp, sz]
        L.psg_set_option.argtypes = [vp, ip, C.c_double]
        L.psg_last_launches.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.psg_version.restype = C.c_char_p
        L.psg_factor_wait.argtypes = [vp, C.POINTER(C.c_double)]
        L.psg_reduced_rhs.argtypes = [vp, vp, vp, ip, vp, cp, sz]
        L.psg_local_factor.argtypes = [C.POINTER(_Block), ip, C.c_double, vp, C.POINTER(vp), cp, sz]
        L.psg_local_query.argtypes = [vp, C.POINTER(_LocalInfo)]
        L.psg_local_read.argtypes = [vp, ip, vp, sz, cp, sz]
        L.psg_local_condense.argtypes = [vp, vp, vp, vp, cp, sz]
        L.psg_local_backsolve.argtypes = [vp, vp, vp, vp, cp, sz]
        L.psg_local_apply.argtypes = [vp, ip, vp, vp, cp, sz]
        L.psg_local_release.argtypes = [vp]
        L.psg_local_release.restype = None
        L.psg_dense_solve.argtypes = [ip, vp, vp, vp, C.POINTER(C.c_longlong), vp, cp, sz]
        _lib = L
    return _lib


def _check(rc: int, err) -> None:
    if rc:
        raise Error(rc - 1, err.value.decode(errors="replace"))


def _is_cuda(t) -> bool:
    return hasattr(t, "is_cuda") and bool(t.is_cuda)


def _addr(t):
    if t is None:
        return None
    if _is_cuda(t):
        return C.c_void_p(t.data_ptr())
    if hasattr(t, "data_ptr") and not isinstance(t, np.ndarray):  # host torch tensor
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)


_raw_stream = None  # torch's current-stream query, cached once CUDA is initialised


def _ptr_of(t):
    if t is None:
        return 0
    if hasattr(t, "data_ptr") and not isinstance(t, np.ndarray):
        return t.data_ptr()
    return t.ctypes.data


def _stream_ptr(stream):
    global _raw_stream
    if stream is None:
        if _raw_stream is not None:
            return C.c_void_p(_raw_stream())
        try:
            import torch
            if torch.cuda.is_available() and torch.cuda.is_initialized():
                getraw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
                if getraw is not None:
                    _raw_stream = lambda: getraw(torch.cuda.current_device())  # noqa: E731
                else:
                    _raw_stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
                return C.c_void_p(_raw_stream())
        except Exception:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


@dataclass
class StructuredMatrix:
    """parsol::StructuredMatrix (structmat.hpp:33-55): compact storage of one
    of the five kinds.  `data`/`corner` may be numpy (host) or CUDA tensors."""
    kind: int
    n: int
    m: int
    s: int
    r: int
    data: Any
    corner: Any = None
    corner_rows: int = 0
    corner_cols: int = 0

    def __post_init__(self):
        if isinstance(self.data, np.ndarray):
            self.data = np.ascontiguousarray(self.data, dtype=np.float64)
        if isinstance(self.corner, np.ndarray):
            self.corner = np.ascontiguousarray(self.corner, dtype=np.float64)

    @property
    def on_device(self) -> bool:
        return _is_cuda(self.data)

    def desc(self) -> _Desc:
        # cached while the storage stays the same (refactor loops call this per step)
        key = (id(self.data), id(self.corner), self.kind, self.n, self.m, self.s, self.r, self.corner_rows,
               self.corner_cols, _ptr_of(self.data), _ptr_of(self.corner))
        c = self.__dict__.get("_desc_cache")
        if c is not None and c[0] == key:
            return c[1]
        n_data = int(self.data.numel() if hasattr(self.data, "numel") else self.data.size)
        d = _Desc(int(self.kind), self.n, self.m, self.s, self.r, _addr(self.data), n_data,
                  _addr(self.corner), self.corner_rows, self.corner_cols, 1 if self.on_device else 0)
        self.__dict__["_desc_cache"] = (key, d)
        return d


@dataclass
class ParallelFactorization:
    """parsol::ParallelFactorization (parfact.hpp:35-46): device handle plus
    the host-side plan / reduced-system metadata."""
    handle: C.c_void_p
    A: StructuredMatrix
    p: int
    strategy: int
    q: int = 0
    dim: int = 0
    k: int = 0
    has_corner: bool = False
    _alive: bool = field(default=True, repr=False)

    def close(self):
        if self._alive and self.handle:
            lib().psg_release(self.handle)
        self._alive = False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, option: str, value: float):
        code = {"speculative": 0, "halo": 1, "cert_tol": 2, "body_cert": 3}[option]
        _check(lib().psg_set_option(self.handle, code, float(value)), C.create_string_buffer(b"bad option"))

    def launches(self):
        f, s = C.c_int(), C.c_int()
        lib().psg_last_launches(self.handle, C.byref(f), C.byref(s))
        return f.value, s.value

    def reduced_blocks(self):
        """Tridiagonal reduced matrix T as (sub, diag, super) host arrays."""
        kk = self.k * self.k
        d = np.empty(self.q * kk)
        sb = np.empty(self.q * kk)
        sp = np.empty(self.q * kk)
        err = C.create_string_buffer(512)
        _check(lib().psg_reduced_blocks(self.handle, d.ctypes.data, sb.ctypes.data, sp.ctypes.data, err, 512), err)
        return sb, d, sp

    def reduced_layout(self):
        """ReducedSystem positions and block sizes, position order (psg_reduced_layout)."""
        pos = np.empty(self.q, np.int32)
        size = np.empty(self.q, np.int32)
        lib().psg_reduced_layout(self.handle, pos.ctypes.data, size.ctypes.data)
        return pos, size

    def reduced_rhs(self, f, stream=None):
        """Reduced right-hand side of f on the reference plan (psg_reduced_rhs):
        f at the separators plus the partitions' condensed contributions."""
        dev = _is_cuda(f)
        if dev:
            import torch
            out = torch.empty(self.dim, dtype=torch.float64, device=f.device)
        else:
            f = np.ascontiguousarray(f, np.float64)
            out = np.empty(self.dim)
        _check_vec(f, self.A.n, "rhs")
        err = C.create_string_buffer(512)
        _check(lib().psg_reduced_rhs(self.handle, _addr(f), _addr(out), 1 if dev else 0, _stream_ptr(stream), err,
                                     512), err)
        return out

    def reduced_dense(self):
        """Dense image of the reduced matrix T (psg_reduced_dense)."""
        T = np.empty((self.dim, self.dim))
        err = C.create_string_buffer(512)
        _check(lib().psg_reduced_dense(self.handle, T.ctypes.data, err, 512), err)
        return T

    def solve(self, f, x=None, stats: SolveStats | None = None, stream=None):
        return solve(self, f, stats=stats, x=x, stream=stream)

    def _errbuf(self):
        e = self.__dict__.get("_err")
        if e is None:
            e = self.__dict__["_err"] = C.create_string_buffer(512)
        return e

    def refactor(self, A: "StructuredMatrix | None" = None, stream=None):
        """New values, same structure (psg_refactor): refactor in place."""
        A = self.A if A is None else A
        d = A.desc()
        err = self._errbuf()
        _check(lib().psg_refactor(self.handle, C.byref(d), _stream_ptr(stream), err, 512), err)
        self.A = A
        return self

    def solve_async(self, f, x, timing: bool = False, stream=None):
        """Enqueue a device solve; x is final after sync() (psg_solve_async)."""
        if not (_is_cuda(f) and _is_cuda(x)):
            raise Error(Errc.InvalidParameter, "solve_async takes device tensors")
        _check_vec(f, self.A.n, "rhs")
        _check_vec(x, self.A.n, "solution")
        err = self._errbuf()
        _check(lib().psg_solve_async(self.handle, _addr(f), _addr(x), 1 if timing else 0, _stream_ptr(stream),
                                     err, 512), err)
        return x

    def sync(self, stats: SolveStats | None = None):
        err = C.create_string_buffer(512)
        _check(lib().psg_sync(self.handle, C.byref(stats) if stats is not None else None, err, 512), err)


def _check_vec(v, n: int, what: str):
    """The reference throws DimensionMismatch for a wrong-length rhs
    (src/parfact.cpp:188); a short, non-fp64 or strided buffer would also be
    read out of bounds by the C ABI, so those are rejected the same way."""
    if v is None:
        return
    if _is_cuda(v) or (hasattr(v, "data_ptr") and not isinstance(v, np.ndarray)):
        import torch
        ok_type = v.dtype == torch.float64
        numel, contig = int(v.numel()), bool(v.is_contiguous())
    else:
        ok_type = v.dtype == np.float64
        numel, contig = int(v.size), bool(v.flags["C_CONTIGUOUS"])
    if not ok_type:
        raise Error(Errc.DimensionMismatch, f"{what}: float64 required, got {v.dtype}")
    if numel != n:
        raise Error(Errc.DimensionMismatch, f"{what} length {numel}, expected {n}")
    if not contig:
        raise Error(Errc.DimensionMismatch, f"{what} must be contiguous")


def parallel_factor(A: StructuredMatrix, p: int, strategy: int = Strategy.Lu, tol: float = 1e-8,
                    stream=None) -> ParallelFactorization:
    d = A.desc()
    h = C.c_void_p()
    err = C.create_string_buffer(1024)
    _check(lib().psg_factor(C.byref(d), int(p), int(strategy), float(tol), _stream_ptr(stream), C.byref(h),
                            err, 1024), err)
    F = ParallelFactorization(h, A, int(p), int(strategy))
    q, dim, k, hc = (C.c_int() for _ in range(4))
    lib().psg_reduced_info(h, C.byref(q), C.byref(dim), C.byref(k), C.byref(hc))
    F.q, F.dim, F.k, F.has_corner = q.value, dim.value, k.value, bool(hc.value)
    return F


def solve(F: ParallelFactorization, f, stats: SolveStats | None = None, x=None, stream=None):
    """Three-phase solve; returns x (same residency as f)."""
    dev = _is_cuda(f)
    if not dev and isinstance(f, (list, tuple)):
        f = np.asarray(f, np.float64)
    if x is None:
        if dev:
            import torch
            x = torch.empty_like(f)
        else:
            f = np.ascontiguousarray(f, np.float64)
            x = np.empty_like(f)
    _check_vec(f, F.A.n, "rhs")
    _check_vec(x, F.A.n, "solution")
    if _is_cuda(x) != dev:
        raise Error(Errc.InvalidParameter, "f and x must both be device or both be host buffers")
    err = C.create_string_buffer(1024)
    st = stats if stats is not None else None
    _check(lib().psg_solve(F.handle, _addr(f), _addr(x), 1 if dev else 0, _stream_ptr(stream),
                           C.byref(st) if st is not None else None, err, 1024), err)
    return x


def solve_reduced(F: ParallelFactorization, rhs, stats: SolveStats | None = None, stream=None):
    dev = _is_cuda(rhs)
    if dev:
        import torch
        x = torch.empty_like(rhs)
    else:
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.empty_like(rhs)
    _check_vec(rhs, F.dim, "reduced rhs")
    err = C.create_string_buffer(1024)
    _check(lib().psg_solve_reduced(F.handle, _addr(rhs), _addr(x), 1 if dev else 0, _stream_ptr(stream),
                                   C.byref(stats) if stats is not None else None, err, 1024), err)
    return x


def residual(A: StructuredMatrix, x, f, stream=None) -> float:
    """||A x - f||_inf / ||f||_inf on the GPU (parfact.cpp:241-251 semantics)."""
    if not _is_cuda(x):
        x, f = np.ascontiguousarray(x, np.float64), np.ascontiguousarray(f, np.float64)
    _check_vec(x, A.n, "residual x")
    _check_vec(f, A.n, "residual f")
    d = A.desc()
    out = C.c_double()
    err = C.create_string_buffer(1024)
    _check(lib().psg_residual(C.byref(d), _addr(x), _addr(f), 1 if _is_cuda(x) else 0, _stream_ptr(stream),
                              C.byref(out), err, 1024), err)
    return out.value


def matvec(A: StructuredMatrix, x, y, stream=None):
    d = A.desc()
    err = C.create_string_buffer(1024)
    _check(lib().psg_matvec(C.byref(d), _addr(x), _addr(y), 1, _stream_ptr(stream), err, 1024), err)
    return y


def plan_partition(A: StructuredMatrix, p: int):
    d = A.desc()
    bb = (C.c_int * p)()
    be = (C.c_int * p)()
    ss = (C.c_int * (p + 1))()
    cnt, k = C.c_int(), C.c_int()
    err = C.create_string_buffer(512)
    _check(lib().psg_plan(C.byref(d), p, bb, be, ss, C.byref(cnt), C.byref(k), err, 512), err)
    return dict(body_ranges=[(bb[i], be[i]) for i in range(p)], separator_starts=list(ss[:cnt.value]),
                sep_size=k.value)


def config_shape(cfg: int, size: int) -> dict:
    k, n, m, s, r, cr, cc = (C.c_int() for _ in range(7))
    ln = C.c_size_t()
    rc = lib().psg_config_shape(cfg, size, C.byref(k), C.byref(n), C.byref(m), C.byref(s), C.byref(r),
                                C.byref(ln), C.byref(cr), C.byref(cc))
    if rc:
        raise Error(rc - 1, "unknown config")
    return dict(kind=k.value, n=n.value, m=m.value, s=s.value, r=r.value, data_len=ln.value,
                corner_rows=cr.value, corner_cols=cc.value)


def generate_config(cfg: int, size: int, seed: int, device="cuda", stream=None):
    """Seeded BASELINE config instance generated on the GPU -> (A, f)."""
    import torch
    sh = config_shape(cfg, size)
    data = torch.empty(sh["data_len"], dtype=torch.float64, device=device)
    corner = torch.empty(64, dtype=torch.float64, device=device) if cfg == 4 else None
    f = torch.empty(sh["n"], dtype=torch.float64, device=device)
    err = C.create_string_buffer(512)
    _check(lib().psg_generate_config(cfg, size, seed, _addr(data), _addr(corner), _addr(f), _stream_ptr(stream),
                                     err, 512), err)
    A = StructuredMatrix(sh["kind"], sh["n"], sh["m"], sh["s"], sh["r"], data, corner, sh["corner_rows"],
                         sh["corner_cols"])
    return A, f


# ---------------------------------------------------------------------------
# per-partition local factorizations (LocalFactorization, reference
# include/parsol/localfact.hpp:24-125) -- factored on the device by
# csrc/psg_local.cu, bit-identical to the reference.
# ---------------------------------------------------------------------------
@dataclass
class PartitionBlock:
    """parsol::PartitionBlock (partition.hpp:50-76): the local system M^(i).
    env is L x (env_s + 1 + env_r); b0/c0 are L x k0, b1/c1 L x k1."""
    kind: int
    m: int
    s: int
    r: int
    L: int
    k0: int
    k1: int
    env_s: int
    env_r: int
    env: np.ndarray
    b0: np.ndarray
    c0: np.ndarray
    b1: np.ndarray
    c1: np.ndarray
    a_right: np.ndarray

    def __post_init__(self):
        for name in ("env", "b0", "c0", "b1", "c1", "a_right"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), np.float64))


_LF = {"fac": 0, "dvec": 1, "z": 2, "w": 3, "y": 4, "v": 5, "alpha1": 6, "alpha2": 7, "beta": 8, "gamma": 9,
       "kept": 10, "cr_elim_idx": 11, "cr_elim_mat": 12, "cr_d2": 13, "cr_d2inv": 14, "cr_cmat": 15,
       "cr_rmat_d2inv": 16, "wmid": 17, "lmat": 18, "linv": 19, "a_order": 20, "kept_rows": 21, "kept_cols": 22,
       "extra_pos": 23, "extra_alpha": 24}


class LocalFactorization:
    """parsol::LocalFactorization on the device; fields are read back on demand."""

    def __init__(self, handle, block: PartitionBlock):
        self.handle = handle
        self.block = block
        info = _LocalInfo()
        lib().psg_local_query(handle, C.byref(info))
        self.info = {k: (list(getattr(info, k)) if k == "rem" else getattr(info, k)) for k, _ in info._fields_}
        self.L, self.k0, self.k1 = info.L, info.k0, info.k1
        self.cr_levels = info.cr_levels
        self.kept_dim = info.k0 + info.k1 + info.n_extras

    def __del__(self):
        try:
            if self.handle:
                lib().psg_local_release(self.handle)
        except Exception:
            pass
        self.handle = None

    def read(self, name: str, count: int, dtype=np.float64):
        out = np.zeros(max(count, 0), dtype)
        if count > 0:
            err = C.create_string_buffer(512)
            _check(lib().psg_local_read(self.handle, _LF[name], out.ctypes.data, out.size, err, 512), err)
        return out

    def field(self, name: str) -> np.ndarray:
        L, k0, k1, i = self.L, self.k0, self.k1, self.info
        kd = self.kept_dim
        shapes = {"z": (L, k0), "w": (L, k0), "y": (L, k1), "v": (L, k1), "alpha1": (k0, k0), "alpha2": (k1, k1),
                  "beta": (k1, k0), "gamma": (k0, k1), "kept": (kd, kd), "dvec": (L if i["strategy"] == 1 else 0,),
                  "fac": ((L, i["env_s"] + 1 + i["env_r"]) if i["core"] == 1 else (0,)),
                  "extra_pos": (i["n_extras"],), "extra_alpha": (i["n_extras"],)}
        shape = shapes[name]
        out = self.read(name, int(np.prod(shape)), np.int32 if name == "extra_pos" else np.float64)
        return out.reshape(shape)

    def _errbuf(self):
        return C.create_string_buffer(512)

    def condense(self, f_body):
        f_body = np.ascontiguousarray(f_body, np.float64)
        _check_vec(f_body, self.L, "condense rhs")
        ghat, kr = np.empty(self.L), np.empty(self.kept_dim)
        err = self._errbuf()
        _check(lib().psg_local_condense(self.handle, f_body.ctypes.data, ghat.ctypes.data, kr.ctypes.data, err,
                                        512), err)
        return ghat, kr

    def backsolve(self, ghat, x_kept):
        ghat = np.ascontiguousarray(ghat, np.float64)
        x_kept = np.ascontiguousarray(x_kept, np.float64)
        _check_vec(ghat, self.L, "ghat")
        _check_vec(x_kept, self.kept_dim, "x_kept")
        x = np.empty(self.L)
        err = self._errbuf()
        _check(lib().psg_local_backsolve(self.handle, ghat.ctypes.data, x_kept.ctypes.data, x.ctypes.data, err,
                                         512), err)
        return x

    def _apply(self, which, rhs):
        rhs = np.ascontiguousarray(rhs, np.float64)
        _check_vec(rhs, self.L, "apply rhs")
        out = np.empty(self.L)
        err = self._errbuf()
        _check(lib().psg_local_apply(self.handle, which, rhs.ctypes.data, out.ctypes.data, err, 512), err)
        return out

    def apply_N_inv(self, rhs):
        return self._apply(0, rhs)

    def apply_S_inv(self, rhs):
        return self._apply(1, rhs)


def factor(strategy: int, block: PartitionBlock, tol: float = 1e-8) -> LocalFactorization:
    """parsol::factor (localfact.hpp:118-125) on the device."""
    b = block
    ptr = lambda a: C.c_void_p(a.ctypes.data) if a.size else None  # noqa: E731
    desc = _Block(int(b.kind), b.m, b.s, b.r, b.L, b.k0, b.k1, b.env_s, b.env_r, ptr(b.env), ptr(b.b0),
                  ptr(b.c0), ptr(b.b1), ptr(b.c1), ptr(b.a_right))
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    _check(lib().psg_local_factor(C.byref(desc), int(strategy), float(tol), None, C.byref(h), err, 512), err)
    return LocalFactorization(h, block)


def factor_lu(block):
    return factor(Strategy.Lu, block)


def factor_lud(block):
    return factor(Strategy.Lud, block)


def factor_cyclic_reduction(block):
    return factor(Strategy.CyclicReduction, block)


def factor_lu_pivot(block, tol):
    return factor(Strategy.LuPivot, block, tol)


def factor_qr(block, tol):
    return factor(Strategy.Qr, block, tol)


def dense_solve(T, rhs):
    """solve_reduced on an explicit reduced matrix T (psg_dense_solve):
    partial-pivot LU on the device, bit-identical to the reference."""
    T = np.ascontiguousarray(T, np.float64)
    rhs = np.ascontiguousarray(rhs, np.float64)
    n = rhs.size
    if T.shape != (n, n):
        raise Error(Errc.DimensionMismatch, "reduced rhs length")
    x = np.empty(n)
    ops = C.c_longlong()
    err = C.create_string_buffer(512)
    _check(lib().psg_dense_solve(n, T.ctypes.data, rhs.ctypes.data, x.ctypes.data, C.byref(ops), None, err, 512),
           err)
    return x, ops.value
