"""CPU checks of the C-ABI library: it loads, exports every function declared
in include/psg.h, and its host-side logic (descriptor validation = make(),
plan_partition, config shapes) matches the reference / oracle.  No compute
call is made (no GPU here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_0912_3678_b200 as psg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "psg.h")).read()
    names = set(re.findall(r"\b(psg_[a-z_]+)\s*\(", hdr))
    assert {"psg_factor", "psg_solve", "psg_release", "psg_residual", "psg_plan"} <= names
    L = psg.lib()
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing
    assert psg.lib().psg_version().startswith(b"psg-b200")


@pytest.mark.parametrize("cfg,size,p", [(0, 4096, 16), (0, 9, 2), (1, 100000, 97), (2, 256, 8), (3, 8192, 16),
                                        (4, 512, 8), (4, 1024, 16)])
def test_plan_matches_oracle(cfg, size, p):
    A, _ = O.generate_config(cfg, size, 1)
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, A.data, A.corner, A.corner_rows, A.corner_cols)
    plan = psg.plan_partition(GA, p)
    ref = O.RefMatrix(A).plan(p) if O.ref_available() else None
    info = O.factor_info(A, p, want_T=False) if size <= 100000 else None
    if ref is not None:
        assert plan["body_ranges"] == ref["body"]
        assert plan["separator_starts"] == ref["seps"]
        assert plan["sep_size"] == ref["k"]
    if info is not None:
        assert len(plan["separator_starts"]) == info["q"]


def test_config_shapes_match_oracle():
    for cfg, size in [(0, 1 << 20), (1, 1 << 26), (2, 1 << 20), (3, 1 << 24), (4, 1 << 18)]:
        assert psg.config_shape(cfg, size) == O.config_shape(cfg, size)


def _err(desc_kwargs, p=4):
    data = np.zeros(desc_kwargs.pop("len"))
    A = psg.StructuredMatrix(data=data, **desc_kwargs)
    with pytest.raises(psg.Error) as e:
        psg.plan_partition(A, p)
    return e.value.code


def test_validation_mirrors_make():
    K = psg.Kind
    assert _err(dict(kind=K.Banded, n=10, m=1, s=1, r=1, len=27)) == psg.Errc.DimensionMismatch
    assert _err(dict(kind=K.Banded, n=3, m=1, s=2, r=1, len=7)) == psg.Errc.InvalidBandwidth
    assert _err(dict(kind=K.BlockTridiagonal, n=12, m=4, s=2, r=1, len=112)) == psg.Errc.InvalidBandwidth
    assert _err(dict(kind=K.Banded, n=10, m=1, s=1, r=1, len=28, corner_rows=1, corner_cols=1)) == \
        psg.Errc.CornerForbidden
    assert _err(dict(kind=K.Banded, n=10, m=1, s=1, r=1, len=28), p=1) == psg.Errc.TooManyPartitions
    assert _err(dict(kind=K.Banded, n=10, m=1, s=1, r=1, len=28), p=6) == psg.Errc.TooManyPartitions
    # the BVP layout s = m, r = 0 is accepted for Babd (make() rejects it; SURVEY.md finding 4)
    A, _ = O.generate_config(4, 64, 1)
    GA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, A.data, A.corner, 8, 8)
    assert len(psg.plan_partition(GA, 4)["separator_starts"]) == 5
