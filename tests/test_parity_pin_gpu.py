"""Parity pinned at the level the data supports.

* every BASELINE config at full size against the C restatement of the
  reference's solve_sequential (bit-identical to the reference,
  tests/test_oracle.py), config 0 also against the unmodified reference's
  parallel_factor + solve at its own p = 1024;
* config 4 against the unmodified reference at N = 2^12, p = 64 (its full N is
  O(N^2) in the reference), with the reference's own parallel-vs-sequential
  spread as the yardstick;
* configs 1-3 at the CONFIG p (65536 / 16384 / 32768): for sampled partitions
  the reference's factor_lu(extract_block(A, plan, i)) alpha1 / alpha2 / beta
  / gamma and condensed kept_rhs (src/localfact.cpp:182-225, 765-781) against
  the GPU's reduced blocks and reduced right-hand side (psg_reduced_blocks,
  psg_reduced_rhs; src/parfact.cpp:89-127, 205-214 assembly);
* CyclicReduction against the reference's strategy 2.

Every achieved value goes to profiles/r02_parity.json (and gpurun_out/), and
each bound below is at most 10x the value measured on the B200 (or the
north-star bound where that is tighter).
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_0912_3678_b200 as psg

from conftest import record_parity

pytestmark = pytest.mark.gpu


def _elem_rel(got, want):
    """largest elementwise relative difference over entries with |want| > 1e-3 max|want|"""
    big = np.abs(want) > 1e-3 * np.max(np.abs(want))
    return float(np.max(np.abs(got[big] - want[big]) / np.abs(want[big])))


def _host(A):
    return O.Matrix(A.kind, A.n, A.m, A.s, A.r, A.data.cpu().numpy(),
                    None if A.corner is None else A.corner.cpu().numpy(), A.corner_rows, A.corner_cols)


CFG = {0: (1 << 20, 1024), 1: (1 << 26, 65536), 2: (1 << 20, 16384), 3: (1 << 24, 32768), 4: (1 << 18, 4096)}
# bounds: north star (1e-12 rel. diff, 1e-13 residual) or 10x the measured value, whichever is tighter
REL_BOUND = {0: 1e-12, 1: 1e-12, 2: 1e-12, 3: 1e-12, 4: 5e-11}  # cfg 4 measured 1.67e-11 (x up to 30)
RES_BOUND = {0: 1e-13, 1: 1e-13, 2: 1e-13, 3: 1e-13, 4: 1e-13}


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_full_size_against_reference_sequential(cuda, cfg):
    size, p = CFG[cfg]
    A, f = psg.generate_config(cfg, size, cfg + 1)
    F = psg.parallel_factor(A, p)
    st = psg.SolveStats()
    x = psg.solve(F, f, st)
    res = psg.residual(A, x, f)
    Ah = _host(A)
    fh = f.cpu().numpy()
    want = O.solve_sequential(Ah, fh)
    xh = x.cpu().numpy()
    rel = O.rel_err(xh, want)
    rec = {"n": A.n, "p": p, "rel_diff_vs_ref_sequential": rel, "elementwise_rel_diff": _elem_rel(xh, want),
           "residual_gpu": res, "residual_ref_sequential": O.residual(Ah, want, fh), "certificate": st.certificate,
           "speculative": st.speculative, "fallbacks": st.fallbacks}
    if cfg == 0 and O.ref_available():  # the reference's own parallel path at the config p
        R = O.RefMatrix(Ah)
        xr, _, _ = R.factor(p).solve(fh)
        rec["rel_diff_vs_ref_parallel_p1024"] = O.rel_err(xh, xr)
        rec["ref_parallel_vs_sequential"] = O.rel_err(xr, want)
        assert rec["rel_diff_vs_ref_parallel_p1024"] <= REL_BOUND[0]
    record_parity(f"cfg{cfg}_full", rec)
    assert rel <= REL_BOUND[cfg]
    assert res <= RES_BOUND[cfg]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [5, 11])
def test_cfg4_against_unmodified_reference(cuda, seed):
    """BASELINE.md's config-4 reference run: the unmodified parallel_factor +
    solve at N = 2^12, p = 64 (and its solve_sequential); the GPU chain path
    must sit within 10x of the reference's own parallel-vs-sequential spread."""
    torch = cuda
    N, p = 1 << 12, 64
    A, f = O.generate_config(4, N, seed)
    R = O.RefMatrix(A)
    xr, _, _ = R.factor(p).solve(f)
    xs = R.solve_sequential(f)
    spread = O.rel_err(xr, xs)
    dev = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, dev(A.data), dev(A.corner), A.corner_rows, A.corner_cols)
    F = psg.parallel_factor(GA, p)
    st = psg.SolveStats()
    x = psg.solve(F, dev(f), st).cpu().numpy()
    d_par, d_seq = O.rel_err(x, xr), O.rel_err(x, xs)
    record_parity(f"cfg4_N4096_p64_seed{seed}", {
        "ref_parallel_vs_ref_sequential": spread, "gpu_vs_ref_parallel": d_par, "gpu_vs_ref_sequential": d_seq,
        "residual_gpu": O.residual(A, x, f), "residual_ref_parallel": R.residual(xr, f),
        "residual_ref_sequential": R.residual(xs, f), "certificate": st.certificate})
    assert max(d_par, d_seq) <= 10 * max(spread, 1e-15)
    assert O.residual(A, x, f) <= 1e-13


def _samples(p, count=24):
    base = np.unique(np.linspace(1, p - 2, count).astype(int))
    return [int(i) for i in base]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_config_p_partition_blocks_match_reference(cuda, cfg):
    """At the config p: reduced-matrix blocks and reduced rhs of sampled
    partition pairs (i, i+1) against the reference's local factorizations."""
    size, p = CFG[cfg]
    A, f = psg.generate_config(cfg, size, cfg + 1)
    F = psg.parallel_factor(A, p)
    F.set_option("speculative", 0)  # the exact reduced matrix (the reference's T)
    sub, diag, sup = F.reduced_blocks()
    rr = F.reduced_rhs(f).cpu().numpy()
    k = F.k
    kk = k * k
    Ah = _host(A)
    fh = f.cpu().numpy()
    R = O.RefMatrix(Ah)
    plan = R.plan(p)
    errs = {"beta": 0.0, "gamma": 0.0, "alpha": 0.0, "rhs": 0.0}
    scale = {"beta": 0.0, "gamma": 0.0, "alpha": 0.0, "rhs": 0.0}

    def local(i):
        blk = O.ref_extract_block(R, p, i)
        lf = O.RefLocal(blk, 0)
        b, e = plan["body"][i - 1]
        _, kept = lf.op(0, fh[b:e])
        get = lambda fid, n: lf.field(fid, n)  # noqa: E731
        return dict(k0=blk["k0"], k1=blk["k1"], a1=get(6, kk), a2=get(7, kk), be=get(8, kk), ga=get(9, kk),
                    kept=kept)

    for i in _samples(p):
        L1, L2 = local(i), local(i + 1)
        s = i - 1  # separator between partitions i and i+1 (0-based)
        pairs = [("beta", L1["be"], sub[s * kk:(s + 1) * kk]) if L1["k0"] else None,
                 ("gamma", L2["ga"], sup[s * kk:(s + 1) * kk]),
                 ("alpha", L1["a2"] + L2["a1"], diag[s * kk:(s + 1) * kk])]
        want_rhs = fh[plan["seps"][s]:plan["seps"][s] + k] + L1["kept"][L1["k0"]:] + L2["kept"][:k]
        pairs.append(("rhs", want_rhs, rr[s * k:(s + 1) * k]))
        for item in pairs:
            if item is None:
                continue
            name, want, got = item
            errs[name] = max(errs[name], float(np.max(np.abs(np.asarray(got) - np.asarray(want)))))
            scale[name] = max(scale[name], float(np.max(np.abs(want))))
    rel = {kname: errs[kname] / scale[kname] if scale[kname] > 0 else errs[kname] for kname in errs}
    record_parity(f"cfg{cfg}_config_p_blocks", {"p": p, "k": k, "partitions_sampled": 2 * len(_samples(p)),
                                           "rel_diff": rel, "scale": scale})
    for kname, v in rel.items():
        assert v <= 1e-13, (kname, v)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,n,m,p,seed", [(0, 1 << 20, 1, 1024, 1), (0, 4000, 1, 16, 3), (1, 4 * 512, 4, 16, 7),
                                             (1, 3 * 300, 3, 10, 8)])
def test_cyclic_reduction_against_reference_strategy_cr(cuda, kind, n, m, p, seed):
    """Strategy CyclicReduction (reference strategy 2, src/localfact.cpp:266-384)
    -- the GPU runs it on the Lu kernels -- against the reference's own CR
    factorization: solution and reduced matrix T."""
    torch = cuda
    if kind == 0 and n == 1 << 20:
        A, f = O.generate_config(0, n, seed)
    else:
        A = O.generate_random(kind, n, m, 1, 1, seed, 2.0)
        f = O.random_vector(n, seed + 1)
    R = O.RefMatrix(A)
    RF = R.factor(p, 2)
    xr, _, _ = RF.solve(f)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, dev(A.data))
    F = psg.parallel_factor(GA, p, psg.Strategy.CyclicReduction)
    x = psg.solve(F, dev(f)).cpu().numpy()
    d = O.rel_err(x, xr)
    rec = {"n": n, "p": p, "gpu_vs_ref_cr": d, "residual_gpu": O.residual(A, x, f), "residual_ref_cr": R.residual(xr, f)}
    _, dim = RF.dims()
    if dim <= 4096:
        Tr = RF.T()
        Tg = F.reduced_dense()
        rec["T_rel_diff"] = float(np.max(np.abs(Tg - Tr)) / np.max(np.abs(Tr)))
        assert rec["T_rel_diff"] <= 1e-13
    record_parity(f"cr_kind{kind}_n{n}_p{p}", rec)
    assert d <= 1e-12
    assert rec["residual_gpu"] <= 1e-13
