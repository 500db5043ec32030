"""Timeline of one config-4 step from %globaltimer stamps (needs the instrumented
build build/prof/libpsg_TL.so copied over libpsg.so; scratch tool)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0912_3678_b200 as psg

A, f = psg.generate_config(4, 1 << 18, 5)
x = torch.empty_like(f)
F = psg.parallel_factor(A, 4096)
lib = ctypes.CDLL(os.path.join(os.path.dirname(psg.__file__), "libpsg.so"))
buf = np.zeros((16, 4), dtype=np.uint64)
names = ["fc2", "down0", "solve1", "down1", "solve2", "fc2-L2-arrival"]
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
    print(f"--- step {it}")
    r = lambda k, j: (t[k, j] - t0) / 1e3
    print(f"  fc2 end {r(0,1):.1f}")
    for sel, k in ((0, 1), (1, 3)):
        print(f"  down{sel}: wait-return {r(k,0):.1f}  staged {r(6+sel,0):.1f}  top solved {r(6+sel,1):.1f}  upper walks {r(6+sel,2):.1f}  end {r(k,1):.1f}")
