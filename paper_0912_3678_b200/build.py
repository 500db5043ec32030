"""In-tree build of the native libraries (sm_100a only).

    libpsg.so          CUDA kernels + the C ABI (include/psg.h)
    libparsol_b200.so  C++ host API mirroring the reference headers
                       (include/parsol/*.hpp) on top of libpsg.so
    psg                command-line tool (generate / solve / verify / plan /
                       bench with STRUCTMAT / VEC files), cli/psg.cpp

Run ``python -m paper_0912_3678_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
INCLUDE = os.path.join(ROOT, "include")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
           "-Xptxas", "-warn-spills"]

# translation units of libpsg.so: the solver (psg_capi.cu includes every
# kernel header) and the per-partition LocalFactorization engine, compiled
# without FMA contraction so its results are the reference's bit for bit.
UNITS = [("psg_capi.cu", []), ("psg_local.cu", ["--fmad=false"])]
OBJDIR = os.path.join(ROOT, "build", "obj")

LIBPSG = os.path.join(PKG, "libpsg.so")
LIBHOST = os.path.join(PKG, "libparsol_b200.so")
CLI = os.path.join(PKG, "psg")
CUDA_HOME = os.path.dirname(os.path.dirname(NVCC))


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _sources(d, exts):
    if not os.path.isdir(d):
        return []
    return sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith(exts))


def source_hash() -> str:
    """sha256 (first 12 hex digits) of every source compiled into libpsg.so;
    psg_version() reports it so a tested binary can be tied to its sources."""
    import hashlib

    h = hashlib.sha256()
    for p in _sources(CSRC, (".cu", ".cuh")) + [os.path.join(INCLUDE, "psg.h")]:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:12]


def build(verbose: bool = True, force: bool = False, ptxas_verbose: bool = False) -> None:
    deps = _sources(CSRC, (".cu", ".cuh")) + [os.path.join(INCLUDE, "psg.h")]
    if force or _newer(LIBPSG, deps):
        extra = ["-Xptxas", "-v"] if ptxas_verbose else []
        objs = []
        os.makedirs(OBJDIR, exist_ok=True)
        for src, flags in UNITS:
            obj = os.path.join(OBJDIR, os.path.basename(src).replace(".cu", ".o"))
            _run([NVCC, *ARCH, *NVFLAGS, *flags, *extra, f"-DPSG_SOURCE_HASH=\"{source_hash()}\"", "-c", "-o", obj,
                  os.path.join(CSRC, src)], verbose)
            objs.append(obj)
        _run([NVCC, *ARCH, "-shared", "-o", LIBPSG, *objs, "-lcuda"], verbose)
    hsrc = _sources(HOST, (".cpp",))
    hdeps = hsrc + _sources(os.path.join(INCLUDE, "parsol"), (".hpp",)) + [LIBPSG]
    if hsrc and (force or _newer(LIBHOST, hdeps)):
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-fopenmp", "-shared", "-I" + INCLUDE, "-o", LIBHOST, *hsrc,
              "-L" + PKG, "-lpsg", "-Wl,-rpath,$ORIGIN"], verbose)
    csrc = _sources(os.path.join(PKG, "cli"), (".cpp",))
    if csrc and (force or _newer(CLI, csrc + [LIBHOST])):
        _run(["g++", "-O2", "-std=c++20", "-I" + INCLUDE, "-I" + os.path.join(CUDA_HOME, "include"), "-o", CLI,
              *csrc, "-L" + PKG, "-lparsol_b200", "-lpsg", "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcudart",
              "-fopenmp", "-Wl,-rpath,$ORIGIN", "-Wl,-rpath," + os.path.join(CUDA_HOME, "lib64")], verbose)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, ptxas_verbose="-v" in sys.argv)
