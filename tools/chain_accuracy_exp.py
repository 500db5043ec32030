import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_0912_3678_b200 as psg
for cfg, size, p in [(4, 1 << 18, 4096), (4, 1 << 14, 256)]:
    for seed in (5, 6):
        A, f = psg.generate_config(cfg, size, seed)
        x = torch.empty_like(f)
        F = psg.parallel_factor(A, p)
        st = psg.SolveStats()
        psg.solve(F, f, st, x=x)
        res = psg.residual(A, x, f)
        print(json.dumps(dict(size=size, seed=seed, nocorr=os.environ.get("PSG_CHAIN_NOCORR"), residual=res, cert=st.certificate, spec=st.speculative, fb=st.fallbacks, xmax=float(x.abs().max()))))
