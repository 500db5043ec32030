"""Step through the chain path on small config-4 instances (debug)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_0912_3678_b200 as psg  # noqa: E402

for size, p in [(127, 4), (1023, 8), (4095, 64)]:
    A, f = O.generate_config(4, size, 3)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, dev(A.data), dev(A.corner), A.corner_rows, A.corner_cols)
    print("factor", size, p, flush=True)
    t = time.time()
    F = psg.parallel_factor(GA, p)
    torch.cuda.synchronize()
    print("  factored", time.time() - t, flush=True)
    st = psg.SolveStats()
    x = psg.solve(F, dev(f), st).cpu().numpy()
    want, _ = O.parallel_solve(A, p, f)
    print("  spec", st.speculative, "fb", st.fallbacks, "cert", st.certificate, "err", O.rel_err(x, want), flush=True)
