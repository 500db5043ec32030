"""Time factor+solve on the full-size BASELINE configs 0-4 (device-resident)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0912_3678_b200 as psg  # noqa: E402

ROOF = {0: 41943024, 1: 2684354544, 2: 469761792, 3: 1207959456, 4: 301991040}
CFG = [(0, 1 << 20, 1024), (1, 1 << 26, 65536), (2, 1 << 20, 16384), (3, 1 << 24, 32768), (4, 1 << 18, 4096)]
peak = 6548.2
sel = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 3, 4]
for cfg, size, p in CFG:
    if cfg not in sel:
        continue
    A, f = psg.generate_config(cfg, size, cfg + 1)
    x = torch.empty_like(f)
    for _ in range(2):
        F = psg.parallel_factor(A, p)
        psg.solve(F, f, x=x)
        F.close()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 5
    st = psg.SolveStats()
    e0.record()
    for _ in range(K):
        F = psg.parallel_factor(A, p)
        psg.solve(F, f, st, x=x)
        F.close()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res = psg.residual(A, x, f)
    n = A.n
    print(json.dumps({"cfg": cfg, "n": n, "p": p, "ms": round(ms, 4), "unknowns_per_s": n / ms * 1e3,
                      "roofline_frac": ROOF[cfg] / (ms * 1e-3) / 1e9 / peak, "residual": res,
                      "cert": st.certificate, "spec": st.speculative,
                      "phases_ms": [round(st.factor_seconds * 1e3, 3), round(st.phase1_seconds * 1e3, 3),
                                    round(st.phase2_seconds * 1e3, 3), round(st.phase3_seconds * 1e3, 3)]}),
          flush=True)
