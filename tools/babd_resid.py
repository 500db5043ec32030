"""Where does the config-4 residual live? max |Ax - f| over BC / separator / body rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_0912_3678_b200 as psg  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
for p in [int(a) for a in sys.argv[2:]] or [4096]:
    A, f = psg.generate_config(4, size, 5)
    F = psg.parallel_factor(A, p)
    st = psg.SolveStats()
    x = psg.solve(F, f, st)
    Ah = O.Matrix(A.kind, A.n, A.m, A.s, A.r, A.data.cpu().numpy(), A.corner.cpu().numpy(), A.corner_rows, A.corner_cols)
    xh, fh = x.cpu().numpy(), f.cpu().numpy()
    r = np.abs(O.matvec(Ah, xh) - fh)
    fn = np.abs(fh).max()
    m = 8
    ss = psg.plan_partition(A, p)["separator_starts"]
    sep = np.zeros(A.n, bool)
    for s0 in ss:
        sep[s0:s0 + m] = True
    print("p", p, "spec", st.speculative, "cert %.2e" % st.certificate, "resid %.2e" % (r.max() / fn),
          "BC %.2e" % (r[:m].max() / fn), "sep %.2e" % (r[sep].max() / fn), "body %.2e" % (r[~sep].max() / fn),
          "|x| %.2e" % np.abs(xh).max(), "|f| %.2e" % fn, flush=True)
