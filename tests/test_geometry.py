"""The layer's n-way chunk decomposition (layer.Geometry): chunks tile the (local expert, capacity
slot) grid exactly once, in the reference's balanced split (core.py:102-105), expert groups first."""

import itertools

import pytest

from paper_2506_22175_b200.layer import Geometry
from paper_2506_22175_b200.spec import balanced_split


@pytest.mark.parametrize("E,N,C,n", [(64, 1, 512, 4), (64, 8, 512, 16), (32, 8, 256, 8), (8, 8, 100, 4),
                                     (64, 1, 80, 3), (12, 2, 7, 5), (64, 1, 512, 1), (4, 4, 9, 9)])
def test_chunks_tile_experts_by_slots(E, N, C, n):
    g = Geometry(T=1, M=64, H=64, E=E, N=N, rank=0, k=1, C=C, n=n)
    e_loc = E // N
    assert g.n_e * g.n_s == n and g.n_e <= e_loc
    assert all(n % d or d > e_loc or d <= g.n_e for d in range(1, n + 1))  # largest divisor <= E_loc
    cover = {}
    for i in range(n):
        ch = g.chunk(i)
        assert ch.part == i % g.n_s and g.rows(i) == N * ch.cs
        for e, s in itertools.product(range(ch.e0, ch.e0 + ch.ne), range(ch.s0, ch.s0 + ch.cs)):
            assert (e, s) not in cover
            cover[(e, s)] = i
    assert len(cover) == e_loc * C
    assert g.group_sizes == balanced_split(e_loc, g.n_e) and g.part_sizes == balanced_split(C, g.n_s)
    # a group's slot parts are consecutive chunks (its weight gradient accumulates over them in order)
    for i in range(n - 1):
        a, b = g.chunk(i), g.chunk(i + 1)
        assert (a.e0 == b.e0 and b.part == a.part + 1) or (b.e0 == a.e0 + a.ne and b.part == 0)
    assert g.max_rows == N * max(g.part_sizes) and g.max_experts == max(g.group_sizes)


def test_expert_split_first():
    # n <= E_loc: pure expert groups, every expert's gradient from one chunk
    g = Geometry(T=1, M=64, H=64, E=64, N=8, rank=0, k=1, C=512, n=4)
    assert (g.n_e, g.n_s) == (4, 1) and [g.chunk(i).ne for i in range(4)] == [2, 2, 2, 2]
    # n > E_loc: groups of one expert, slots split in parts
    g = Geometry(T=1, M=64, H=64, E=64, N=8, rank=0, k=1, C=512, n=16)
    assert (g.n_e, g.n_s) == (8, 2) and g.chunk(1).part == 1 and g.chunk(1).s0 == 256
