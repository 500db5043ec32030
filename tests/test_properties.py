"""SPEC invariants checkable without a GPU: the reduced-size law (q constant
across n at fixed p, p-1 without / p+1 with the corner) through the C ABI plan,
and the TooManyPartitions / p < 2 errors (src/partition.cpp:53,83-85)."""
import pytest

import oracle as O
import paper_0912_3678_b200 as psg


@pytest.mark.parametrize("kind,m,s,r", [(0, 1, 1, 1), (0, 1, 3, 3), (1, 4, 1, 1), (2, 4, 2, 2), (3, 4, 2, 2)])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_reduced_size_law(kind, m, s, r, p):
    qs = []
    for n in (48, 96, 400):
        A = O.generate_random(kind, n, m, s, r, 3, 2.0)
        SA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, A.data, A.corner, A.corner_rows, A.corner_cols)
        plan = psg.plan_partition(SA, p)
        qs.append(len(plan["separator_starts"]))
    assert qs[0] == qs[1] == qs[2] == (p + 1 if kind == 3 else p - 1)


def test_partition_count_errors():
    A = O.generate_random(0, 40, 1, 1, 1, 1, 2.0)
    SA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, A.data)
    for p in (0, 1, 41):
        with pytest.raises(psg.Error) as e:
            psg.plan_partition(SA, p)
        assert e.value.code == psg.Errc.TooManyPartitions
