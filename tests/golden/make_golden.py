"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
/root/reference/proj/src compiled by oracle/Makefile).  Run here, where the
reference is mounted:

    make -C oracle all ref && python tests/golden/make_golden.py

Each fixture stores the reference's own outputs for one seeded instance:
x from parallel_factor(Lu)+solve at the given p, x from solve_sequential,
the phase-2 op count, the residual, the dense reduced matrix T (small dims)
and the alpha/beta/gamma blocks of the first partitions.  The matrix itself is
regenerated from (cfg, size, seed) by the SplitMix64 generator; its SHA-256
is stored to pin the generator.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

CASES = [
    # name, cfg, size, seed, p
    ("cfg0_n4096_p16", 0, 4096, 1, 16),
    ("cfg0_n1e5_p100", 0, 100000, 11, 100),
    ("cfg1_n65536_p64", 1, 65536, 2, 64),
    ("cfg2_N256_p8", 2, 256, 3, 8),
    ("cfg3_n8192_p16", 3, 8192, 4, 16),
    ("cfg4_N512_p8", 4, 512, 5, 8),
    ("cfg4_N1024_p16", 4, 1024, 6, 16),
]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    O.ref_set_threads(1)
    for name, cfg, size, seed, p in CASES:
        A, f = O.generate_config(cfg, size, seed)
        R = O.RefMatrix(A)
        F = R.factor(p)
        x, ops, _ = F.solve(f)
        xs = R.solve_sequential(f)
        res = R.residual(x, f)
        q, dim = F.dims()
        T = F.T() if dim <= 1200 else np.zeros((0, 0))
        plan = R.plan(p)
        out = dict(cfg=cfg, size=size, seed=seed, p=p, kind=A.kind, n=A.n, m=A.m, s=A.s, r=A.r,
                   data_sha=sha(A.data), f_sha=sha(f), x=x, x_seq=xs, reduced_ops=ops, residual=res,
                   q=q, dim=dim, T=T, seps=np.array(plan["seps"]), k=plan["k"],
                   body=np.array(plan["body"]))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(f"{name}: n={A.n} q={q} dim={dim} ops={ops} residual={res:.2e}")
    # SPEC.md known answers, run through the reference
    kat = {}
    T3 = O.Matrix(O.BANDED, 3, 1, 1, 1, np.array([-1.0, -1.0, 2.0, 2.0, 2.0, -1.0, -1.0]))
    kat["toeplitz3_x"] = O.RefMatrix(T3).factor(2).solve(np.ones(3))[0]
    T9 = O.Matrix(O.BANDED, 9, 1, 1, 1, np.concatenate([-np.ones(8), 2 * np.ones(9), -np.ones(8)]))
    kat["toeplitz9_q"] = O.RefMatrix(T9).factor(2).dims()[0]
    I8 = O.Matrix(O.BANDED, 8, 1, 1, 1, np.concatenate([np.zeros(7), np.ones(8), np.zeros(7)]))
    f8 = np.arange(1.0, 9.0)
    kat["identity_x"] = O.RefMatrix(I8).factor(4).solve(f8)[0]
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **kat)
    print("kat:", {k: v for k, v in kat.items()})


if __name__ == "__main__":
    main()
