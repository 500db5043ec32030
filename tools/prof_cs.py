"""Per-CTA phase timeline of the config-4 solve passes (%globaltimer stamps).

Needs a -DPSG_PROF build of libpsg.so (not the shipped one):
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
        --expt-relaxed-constexpr -DPSG_PROF -DPSG_SOURCE_HASH='"prof"' -c -o /tmp/capi.o \
        paper_0912_3678_b200/csrc/psg_capi.cu
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_0912_3678_b200/libpsg.so \
        /tmp/capi.o build/obj/psg_local.o -lcuda
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
for _ in range(3):
    F.refactor(A)
    F.solve_async(f, x)
    F.sync()
torch.cuda.synchronize()
lib = ctypes.CDLL(os.path.join(os.path.dirname(psg.__file__), "libpsg.so"))
buf = np.zeros((2, 1024, 6), dtype=np.int64)
lib.psg_prof_dump(buf.ctypes.data_as(ctypes.c_void_p))
for km in range(2):
    t = buf[km].astype(np.float64)
    t0 = t[:, 0].min()
    d = (t[:, 1:5] - t[:, 0:4]) / 1e3
    print(f"KM{km + 1}: kernel span {(t[:, 4].max() - t0) / 1e3:.1f} us; CTA life mean {((t[:, 4] - t[:, 0]) / 1e3).mean():.1f} us")
    print("   phase means (us): stage %.1f  wait+walk %.1f  run %.1f  up/cert %.1f" % tuple(d.mean(axis=0)))
    print("   phase p90   (us): stage %.1f  wait+walk %.1f  run %.1f  up/cert %.1f" % tuple(np.percentile(d, 90, axis=0)))
    starts = np.sort((t[:, 0] - t0) / 1e3)
    print("   CTA start times (us): p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(starts, [10, 50, 90, 100])))
