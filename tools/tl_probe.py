"""Timeline of one config-4 step from %globaltimer stamps, per kernel.

Needs a -DPSG_PROF build of libpsg.so in place of the shipped one (the stamps
compile to nothing otherwise):
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
        --expt-relaxed-constexpr -DPSG_PROF -DPSG_SOURCE_HASH='"prof"' -c -o build/prof_capi.o \
        paper_0912_3678_b200/csrc/psg_capi.cu
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_0912_3678_b200/libpsg.so \
        build/prof_capi.o build/obj/psg_local.o -lcuda
Times are us from the first chain_fc2 CTA's start.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0912_3678_b200 as psg

A, f = psg.generate_config(4, 1 << 18, 5)
x = torch.empty_like(f)
F = psg.parallel_factor(A, 4096)
lib = ctypes.CDLL(os.path.join(os.path.dirname(psg.__file__), "libpsg.so"))
buf = np.zeros((16, 4), dtype=np.uint64)
for it in range(6):
    torch.cuda.synchronize()
    lib.psg_tl_dump(buf.ctypes.data_as(ctypes.c_void_p), 1)
    F.refactor(A)
    F.solve_async(f, x)
    F.sync()
    torch.cuda.synchronize()
    lib.psg_tl_dump(buf.ctypes.data_as(ctypes.c_void_p), 0)
    if it < 3:
        continue
    t = buf.astype(np.float64)
    t0 = t[0, 0]

    def r(k, j):
        return (t[k, j] - t0) / 1e3

    print(f"--- step {it}")
    print(f"  factor: level 1 done {r(8, 0):.1f} | L2 arrived {r(9, 1):.1f} tree {r(9, 3):.1f} | L3 arrived {r(10, 1):.1f} "
          f"tree {r(10, 3):.1f} | top arrived {r(11, 1):.1f} tree {r(11, 3):.1f} | G built {r(12, 0):.1f} LU {r(12, 1):.1f} "
          f"| end {r(0, 1):.1f}")
    for sel, k in ((0, 1), (1, 3)):
        print(f"  down{sel}: wait-return {r(k, 0):.1f}  staged {r(6 + sel, 0):.1f}  top solved {r(6 + sel, 1):.1f}  "
              f"upper walks {r(6 + sel, 2):.1f}  end {r(k, 1):.1f}")
    for km in (1, 2):
        print(f"  pass{km}: first CTA start {r(2 * km, 0):.1f}  first wait-return {r(2 * km, 2):.1f}  end {r(2 * km, 1):.1f}")
