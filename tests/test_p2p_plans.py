"""CPU tests of the peer-memory exchange plans (comm.pull_plan / push_plan /
signal_plan / reduce_plan): N ranks' windows and expert-side buffers are
numpy byte arrays, the plans' 2-D copies are interpreted on them, and the
result must equal the block layout of comm.block_plan (the one definition
the NCCL path and the oracle's block transpose share).  Flag wiring is
checked as sets: every wait / arrival flag is raised by exactly the peers
that must have finished first.
"""

import numpy as np
import pytest

from paper_2506_22175_b200 import _lib
from paper_2506_22175_b200.comm import (
    FLAG_DWG,
    FLAG_GO_READY,
    FLAG_TI_READY,
    WindowLayout,
    block_plan,
    pull_plan,
    push_plan,
    reduce_plan,
    signal_plan,
)
from paper_2506_22175_b200.spec import balanced_split


def _copy(bufs, plan):
    def at(sym):
        kind, key, off = sym
        return bufs[(kind, key)], off

    for dst, src, dpitch, spitch, width, height in plan["copy"]:
        (db, do), (sb, so) = at(dst), at(src)
        for h in range(height):
            db[do + h * dpitch: do + h * dpitch + width] = sb[so + h * spitch: so + h * spitch + width]


def _flags(plan, key):
    return {(k, r, off) for (k, r, off) in plan[key]}


def _expected_expert_side(N, e_loc, C, c_i, s_i, M, esz, t_i_of, rank, x_stride, x_row0, out):
    """Expert-side bytes of `rank` after chunk i's dispatch, from block_plan's element offsets."""
    for src in range(N):
        peers, soff, roff = block_plan(_lib.A2A_DISPATCH, N, e_loc, c_i, M, C, s_i, x_stride, x_row0)
        # blocks `src` sends to `rank` land at the receive offsets `rank` posts for `src`
        sends = [so for p, so in zip(peers, soff) if p == rank]
        recvs = [ro for p, ro in zip(peers, roff) if p == src]
        for so, ro in zip(sends, recvs):
            out[ro * esz:(ro + c_i * M) * esz] = t_i_of[src][so * esz:(so + c_i * M) * esz]
    return out


@pytest.mark.parametrize("N,e_loc,C,n,M", [(2, 2, 5, 2, 8), (3, 1, 7, 3, 4), (4, 2, 6, 4, 8), (8, 1, 4, 1, 4)])
@pytest.mark.parametrize("full", [True, False])
def test_dispatch_pull_and_combine_push(N, e_loc, C, n, M, full):
    esz = 2
    E = N * e_loc
    L = WindowLayout(N, E, C, M, esz, n, E * M)
    rng = np.random.default_rng(N * 100 + C)
    win = {r: np.zeros(L.total, np.uint8) for r in range(N)}
    for r in range(N):
        win[r][L.off["t_i"]:L.off["t_i"] + E * C * M * esz] = rng.integers(0, 255, E * C * M * esz, dtype=np.uint8)
    t_i_of = {r: win[r][L.off["t_i"]:L.off["t_i"] + E * C * M * esz].copy() for r in range(N)}
    sizes = balanced_split(C, n)
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(int)
    exp_size = e_loc * N * C * M * esz
    expert = {r: np.zeros(exp_size, np.uint8) for r in range(N)}
    want_full = {r: np.zeros(exp_size, np.uint8) for r in range(N)}
    for i, (c_i, s_i) in enumerate(zip(sizes, starts)):
        c_i, s_i = int(c_i), int(s_i)
        x_stride, x_row0 = (N * C, N * s_i) if full else (N * c_i, 0)
        ring = {r: np.zeros(exp_size, np.uint8) for r in range(N)}
        bufs = {("win", r): win[r] for r in range(N)}
        readiness = set()
        for r in range(N):
            readiness |= _flags(signal_plan(L, r, FLAG_TI_READY), "signal")
        for r in range(N):
            target = expert[r] if full else ring[r]
            last = i == len(sizes) - 1
            plan = pull_plan(L, r, e_loc, C, c_i, s_i, "t_i", FLAG_TI_READY, ("loc", r, 0), x_stride, x_row0,
                             reset=last)
            # rank r waits for exactly the N-1 peers' "T_I ready" flags, all of which are raised
            assert len(plan["wait"]) == N - 1 and _flags(plan, "wait") <= readiness
            assert {off for (_, rr, off) in plan["wait"]} == {L.flag(FLAG_TI_READY, p) for p in range(N) if p != r}
            # the last chunk's pull (the step's last wait on them) resets exactly its own waited flags
            assert _flags(plan, "reset") == (_flags(plan, "wait") if last else set())
            assert all(rr == r for (_, rr, _) in plan["reset"])
            # a re-dispatch (RC_i) neither waits nor resets, and moves the same bytes
            re = pull_plan(L, r, e_loc, C, c_i, s_i, "t_i", None, ("loc", r, 0), x_stride, x_row0)
            assert re["wait"] == [] and re["reset"] == [] and re["copy"] == plan["copy"]
            _copy({**bufs, ("loc", r): target}, plan)
            want = _expected_expert_side(N, e_loc, C, c_i, s_i, M, esz, t_i_of, r, x_stride, x_row0,
                                         want_full[r] if full else np.zeros(exp_size, np.uint8))
            np.testing.assert_array_equal(target, want)
        # combine: every expert rank pushes its rows back; owners' T_O must equal the T_I they sent
        # (the identity expert), restricted to chunk i's slots
        raised = {r: set() for r in range(N)}
        for r in range(N):
            src = expert[r] if full else ring[r]
            plan = push_plan(L, r, e_loc, C, c_i, s_i, "t_o", L.r_slot(i), ("loc", r, 0), x_stride, x_row0)
            _copy({**bufs, ("loc", r): src}, plan)
            for (_, d, off) in plan["signal"]:
                raised[d].add(off)
            assert {off for (_, rr, off) in plan["arrive"]} == {L.flag(L.r_slot(i), p) for p in range(N) if p != r}
            assert all(rr == r for (_, rr, _) in plan["arrive"])
            assert plan["reset"] == plan["arrive"]  # the arrival wait is the flags' only wait of the step
        for r in range(N):
            assert raised[r] == {L.flag(L.r_slot(i), p) for p in range(N) if p != r}
            t_o = win[r][L.off["t_o"]:L.off["t_o"] + E * C * M * esz].reshape(E, C, M * esz)
            t_i = t_i_of[r].reshape(E, C, M * esz)
            np.testing.assert_array_equal(t_o[:, s_i:s_i + c_i], t_i[:, s_i:s_i + c_i])


def test_flag_slots_are_disjoint():
    N, n = 4, 3
    L = WindowLayout(N, 8, 5, 16, 2, n, 8 * 16)
    slots = [FLAG_TI_READY, FLAG_GO_READY, FLAG_DWG] + [L.r_slot(i) for i in range(n)] + \
        [L.br_slot(i) for i in range(n)]
    offs = {L.flag(s_, p) for s_ in slots for p in range(N)}
    assert len(offs) == len(slots) * N
    assert min(offs) >= L.off["flags"] and max(offs) + 4 <= L.total
    # the four dispatch-side buffers and the stage never overlap
    spans = sorted((L.off[k], L.off[k] + (8 * 5 * 16 * 2 if k != "stage" else N * L.stage_slice))
                   for k in ("t_i", "t_o", "g_o", "g_i", "stage"))
    for (a0, a1), (b0, _) in zip(spans, spans[1:]):
        assert a1 <= b0


@pytest.mark.parametrize("N", [2, 3, 8])
def test_gate_gradient_reduce_plan(N):
    E, M = 4, 8
    L = WindowLayout(N, E, 2, M, 2, 1, E * M)
    rng = np.random.default_rng(N)
    win = {r: np.zeros(L.total, np.uint8) for r in range(N)}
    slices = {r: rng.standard_normal(E * M).astype(np.float32) for r in range(N)}
    for r in range(N):
        off = L.stage(r)
        win[r][off:off + E * M * 4] = slices[r].view(np.uint8)
    raised = {r: set() for r in range(N)}
    for r in range(N):
        plan = reduce_plan(L, r, E * M * 4)
        _copy({("win", q): win[q] for q in range(N)}, plan)
        for (_, d, off) in plan["signal"]:
            raised[d].add(off)
        assert plan["reset"] == plan["arrive"]
    for r in range(N):
        assert raised[r] == {L.flag(FLAG_DWG, p) for p in range(N) if p != r}
        got = [win[r][L.stage(p):L.stage(p) + E * M * 4].view(np.float32) for p in range(N)]
        for p in range(N):
            np.testing.assert_array_equal(got[p], slices[p])
        # the stride mpm_sum_slices walks: stage(p) = stage(0) + p * stage_slice
        assert all(L.stage(p) - L.stage(0) == p * L.stage_slice for p in range(N))


@pytest.mark.parametrize("N,e_loc,C,e0,ne,s0,cs", [(2, 4, 6, 1, 2, 2, 3), (4, 3, 5, 2, 1, 0, 5), (3, 2, 4, 0, 2, 1, 2)])
def test_expert_group_chunk_plans(N, e_loc, C, e0, ne, s0, cs):
    """A chunk of local experts [e0, e0+ne) x slots [s0, s0+cs) (Geometry.chunk): the peer-memory
    pull lands exactly block_plan's rows, into a ring slot (x_row0 = 0) and into an all-chunk buffer
    (x_row0 = e0*N*C + N*s0), and the push inverts it."""
    M, esz = 4, 2
    E = N * e_loc
    L = WindowLayout(N, E, C, M, esz, 1, E * M)
    rng = np.random.default_rng(N + e0 + cs)
    win = {r: np.zeros(L.total, np.uint8) for r in range(N)}
    for r in range(N):
        win[r][L.off["t_i"]:L.off["t_i"] + E * C * M * esz] = rng.integers(0, 255, E * C * M * esz, dtype=np.uint8)
    t_i_of = {r: win[r][L.off["t_i"]:L.off["t_i"] + E * C * M * esz].copy() for r in range(N)}
    for full in (False, True):
        x_stride, x_row0 = (N * C, e0 * N * C + N * s0) if full else (N * cs, 0)
        size = e_loc * N * C * M * esz
        for r in range(N):
            got = np.zeros(size, np.uint8)
            plan = pull_plan(L, r, e_loc, C, cs, s0, "t_i", FLAG_TI_READY, ("loc", r, 0), x_stride, x_row0,
                             e0=e0, ne=ne)
            assert all(h == ne for (*_, h) in plan["copy"])
            _copy({**{("win", q): win[q] for q in range(N)}, ("loc", r): got}, plan)
            want = np.zeros(size, np.uint8)
            for src in range(N):
                peers, soff, roff = block_plan(_lib.A2A_DISPATCH, N, e_loc, cs, M, C, s0, x_stride, x_row0,
                                               e0=e0, ne=ne)
                sends = [so for p, so in zip(peers, soff) if p == r]
                recvs = [ro for p, ro in zip(peers, roff) if p == src]
                assert len(sends) == len(recvs) == ne
                for so, ro in zip(sends, recvs):
                    want[ro * esz:(ro + cs * M) * esz] = t_i_of[src][so * esz:(so + cs * M) * esz]
            np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("N,e_loc,C,n", [(2, 4, 6, 2), (4, 2, 5, 4), (3, 1, 7, 3), (2, 8, 4, 16)])
def test_fused_push_matches_pull_layout(N, e_loc, C, n):
    """The fused dispatch (push_dispatch_plan, as mpm_dispatch_push executes it: gather through the
    slot-owner map, store into every destination's window) lands every chunk's rows exactly where the
    pull path (block_plan / pull_plan) puts them, with zero rows for unused slots; every source raises
    its flag of the chunk in every peer's window, and the receiver waits for exactly the peers'."""
    from paper_2506_22175_b200.comm import push_dispatch_plan
    from paper_2506_22175_b200.layer import Geometry
    M, esz = 4, 1
    E = N * e_loc
    L = WindowLayout(N, E, C, M, esz, n, E * M, fused=True)
    rng = np.random.default_rng(N * 7 + n)
    T, k = 9, 2
    xs, invs, t_is = {}, {}, {}
    for r in range(N):
        xs[r] = rng.integers(1, 255, (T, M), dtype=np.uint8)
        inv = np.full(E * C, -1, np.int64)
        a = rng.permutation(T * k)[: min(T * k, E * C)]
        cells = rng.choice(E * C, size=len(a), replace=False)
        inv[cells] = a
        invs[r] = inv
        t_i = np.zeros((E * C, M), np.uint8)  # what the pull path's permute would build
        t_i[cells] = xs[r][a // k]
        t_is[r] = t_i.reshape(-1)
    g = Geometry(T=T, M=M, H=M, E=E, N=N, rank=0, k=k, C=C, n=n)
    win = {r: np.zeros(L.total, np.uint8) for r in range(N)}
    want = {r: np.zeros(e_loc * N * C * M, np.uint8) for r in range(N)}
    for i in range(n):
        ch = g.chunk(i)
        raised = {r: set() for r in range(N)}
        for src in range(N):
            plan = push_dispatch_plan(L, src, e_loc, C, ch.cs, ch.s0, "t_di", L.s_slot(i), e0=ch.e0, ne=ch.ne)
            geo = plan["geom"]
            for d, (_, rr, off) in enumerate(plan["dst"]):
                assert rr == d and off == L.off["t_di"]
                for el in range(ch.e0, ch.e0 + ch.ne):
                    for s_ in range(ch.s0, ch.s0 + ch.cs):
                        a = invs[src][(d * e_loc + el) * C + s_]
                        row = (el - geo["e0"]) * geo["x_stride"] + geo["x_row0"] + src * ch.cs + (s_ - ch.s0)
                        val = np.zeros(M, np.uint8) if a < 0 else xs[src][a // k]
                        win[d][off + row * M: off + (row + 1) * M] = val
            for (_, d, off) in plan["flag"]:
                if d != src:
                    raised[d].add(off)
            assert {off for (_, rr, off) in plan["arrive"]} == {L.flag(L.s_slot(i), p) for p in range(N) if p != src}
            assert plan["reset"] == plan["arrive"]
        for r in range(N):
            assert raised[r] == {L.flag(L.s_slot(i), p) for p in range(N) if p != r}
            # the pull path's rows for this chunk (full buffer, block_plan layout)
            x_row0 = ch.e0 * N * C + N * ch.s0
            for src in range(N):
                peers, soff, roff = block_plan(_lib.A2A_DISPATCH, N, e_loc, ch.cs, M, C, ch.s0, N * C, x_row0,
                                               e0=ch.e0, ne=ch.ne)
                sends = [so for p, so in zip(peers, soff) if p == r]
                recvs = [ro for p, ro in zip(peers, roff) if p == src]
                for so, ro in zip(sends, recvs):
                    want[r][ro:ro + ch.cs * M] = t_is[src][so:so + ch.cs * M]
    for r in range(N):
        got = win[r][L.off["t_di"]:L.off["t_di"] + e_loc * N * C * M]
        np.testing.assert_array_equal(got, want[r])
