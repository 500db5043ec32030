"""Print speculative/fallback/certificate for the block spec test shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_0912_3678_b200 as psg  # noqa: E402

SHAPES = [(1, 4 * 4096, 4, 1, 1, 16), (1, 4 * 1000, 4, 1, 1, 7), (1, 3 * 3000, 3, 1, 1, 9), (1, 2 * 5000, 2, 1, 1, 5),
          (0, 20000, 1, 3, 3, 8), (0, 9001, 1, 2, 3, 5), (0, 7000, 1, 2, 2, 6), (0, 12000, 1, 4, 4, 10),
          (0, 8000, 1, 1, 4, 4)]
for dom in (2.0, 4.0):
    for kind, n, m, s, r, p in SHAPES:
        A = O.generate_random(kind, n, m, s, r, 31 + n, dom)
        f = O.random_vector(n, 5)
        want, _ = O.parallel_solve(A, p, f)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, dev(A.data), None, 0, 0)
        F = psg.parallel_factor(GA, p)
        F.set_option("cert_tol", 1.0)
        st = psg.SolveStats()
        x = psg.solve(F, dev(f), st).cpu().numpy()
        print(dom, (kind, n, m, s, r, p), "spec", st.speculative, "fb", st.fallbacks, "cert %.3e" % st.certificate,
              "err %.3e" % O.rel_err(x, want), flush=True)
