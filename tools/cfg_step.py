"""bench-like step (refactor + async solve + sync) on one BASELINE config.

    python tools/cfg_step.py CFG [STEPS]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0912_3678_b200 as psg  # noqa: E402

CFG = {0: (1 << 20, 1024), 1: (1 << 26, 65536), 2: (1 << 20, 16384), 3: (1 << 24, 32768), 4: (1 << 18, 4096)}
ROOF = {0: 41943024, 1: 2684354544, 2: 469761792, 3: 1207959456, 4: 301991040}
cfg = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
size, p = CFG[cfg]
A, f = psg.generate_config(cfg, size, cfg + 1)
x = torch.empty_like(f)
F = psg.parallel_factor(A, p)
if os.environ.get("BODY_CERT"):
    F.set_option("body_cert", 1)
for _ in range(3):
    F.refactor(A)
    F.solve_async(f, x)
    F.sync()
torch.cuda.synchronize()
if os.environ.get("ALONE"):  # bench.py's small-config mode: L2 flushed, each step's device time alone
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f.device)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        flush.random_(0, 255)
        a.record()
        F.refactor(A)
        F.solve_async(f, x)
        b.record()
        F.sync()
    torch.cuda.synchronize()
    print(json.dumps({"cfg": cfg, "alone_ms": round(sum(a.elapsed_time(b) for a, b in evs) / steps, 4)}))
    sys.exit(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = psg.SolveStats()
e0.record()
for _ in range(steps):
    F.refactor(A)
    F.solve_async(f, x, timing=not os.environ.get("NOTIMING"))
F.sync(st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
res = psg.residual(A, x, f)
print(json.dumps({"cfg": cfg, "ms": round(ms, 4), "roofline_frac": round(ROOF[cfg] / (ms * 1e-3) / 1e9 / 6548.2, 4),
                  "residual": res, "cert": st.certificate, "spec": st.speculative,
                  "factor_ms": round(st.factor_seconds * 1e3, 4),
                  "phase_ms": [round(st.phase1_seconds * 1e3 / steps, 4), round(st.phase2_seconds * 1e3 / steps, 4),
                               round(st.phase3_seconds * 1e3 / steps, 4)]}))
