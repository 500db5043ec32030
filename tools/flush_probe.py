"""Per-step device time of the L2-resident configs under different L2 flushes.

    python tools/flush_probe.py [CFG ...]

write:       512 MB written before the step (L2 left full of DIRTY lines: the
             step's first misses also pay their write-back)
write+read:  the same write, then a 512 MB read of another buffer (L2 left
             full of clean lines that belong to neither A, f nor x)
none:        back-to-back steps, inputs L2-warm
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0912_3678_b200 as psg  # noqa: E402

CFG = {0: (1 << 20, 1024), 2: (1 << 20, 16384), 4: (1 << 18, 4096)}
cfgs = [int(a) for a in sys.argv[1:]] or [0, 2, 4]
dev = torch.device("cuda", 0)
wbuf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
rbuf = torch.ones(512 << 18, dtype=torch.float32, device=dev)
sink = torch.zeros(1, dtype=torch.float32, device=dev)


def flush(mode):
    if mode == "none":
        return
    wbuf.random_(0, 255)
    if mode == "write+read":
        sink.copy_(rbuf.sum().reshape(1))


for cfg in cfgs:
    size, p = CFG[cfg]
    A, f = psg.generate_config(cfg, size, cfg + 1)
    x = torch.empty_like(f)
    H = psg.parallel_factor(A, p)
    for _ in range(3):
        H.refactor(A)
        H.solve_async(f, x)
        H.sync()
    for mode in ("write", "write+read", "none", "write", "write+read"):
        steps = 20
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        st = psg.SolveStats()
        for e0, e1 in evs:
            flush(mode)
            e0.record()
            H.refactor(A)
            H.solve_async(f, x)
            e1.record()
            H.sync(st)
        torch.cuda.synchronize()
        t = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
        print(json.dumps({"cfg": cfg, "flush": mode, "mean_us": round(sum(t) / steps * 1e3, 2),
                          "median_us": round(t[steps // 2] * 1e3, 2), "min_us": round(t[0] * 1e3, 2)}), flush=True)
    H.close()
