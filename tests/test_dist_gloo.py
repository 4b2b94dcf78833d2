"""World-size-2 tests of the multi-rank host logic over gloo (CPU).

* the chunk all-to-all block plan (comm.block_plan), executed with real
  torch.distributed point-to-point sends, lands every (source, expert, slot)
  row exactly where the expert-side GEMM view expects it — checked against the
  oracle's own all-to-all (a block transpose) — and combine inverts dispatch;
* Algorithm-1 decisions are rank-symmetric when measurements are reduced with
  the max over ranks (calibrate._max_over_ranks), even with rank-local noise;
* the replicated gate's gradient all-reduce is a sum.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_oracle as O
from paper_2506_22175_b200 import _lib
from paper_2506_22175_b200.comm import block_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        q.put((rank, exc))
    finally:
        dist.destroy_process_group()


def spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def _exchange(plan, src, dst, block):
    peers, soff, roff = plan
    reqs = []
    for peer, so, ro in zip(peers, soff, roff):
        chunk_s = src.view(-1)[so:so + block]
        chunk_r = dst.view(-1)[ro:ro + block]
        if peer == dist.get_rank():
            chunk_r.copy_(chunk_s)
        else:
            reqs.append(dist.isend(chunk_s.contiguous(), peer))
            buf = torch.empty(block, dtype=src.dtype)
            reqs.append((dist.irecv(buf, peer), chunk_r, buf))
    for r in reqs:
        if isinstance(r, tuple):
            r[0].wait()
            r[1].copy_(r[2])
        else:
            r.wait()


def chunk_a2a_case(rank, world):
    """Every chunk of an expert-major [E][C][M] dispatch buffer, exchanged into
    (a) an all-chunk expert-side buffer [E_loc][N*C][M] and (b) a per-chunk
    ring slot [E_loc][N*c_i][M], then combined back."""
    E_loc, C, M, n = 3, 7, 4, 3
    E = E_loc * world
    sizes = O.partition_sizes(C, n)
    starts = O.chunk_starts(C, n)
    src = torch.tensor([[[rank * 10000 + e * 1000 + s * 10 + m for m in range(M)] for s in range(C)]
                        for e in range(E)], dtype=torch.float32)
    full = torch.full((E_loc, world * C, M), -1.0)
    back = torch.full_like(src, -1.0)
    rings = []
    for i in range(n):
        c_i, s_i = sizes[i], starts[i]
        _exchange(block_plan(_lib.A2A_DISPATCH, world, E_loc, c_i, M, C, s_i, world * C, world * s_i),
                  src, full, c_i * M)
        ring = torch.full((E_loc, world * c_i, M), -1.0)
        _exchange(block_plan(_lib.A2A_DISPATCH, world, E_loc, c_i, M, C, s_i, world * c_i, 0), src, ring, c_i * M)
        rings.append(ring.numpy())
        _exchange(block_plan(_lib.A2A_COMBINE, world, E_loc, c_i, M, C, s_i, world * C, world * s_i),
                  full, back, c_i * M)
    return full.numpy(), rings, back.numpy(), src.numpy()


def test_block_plan_dispatch_and_combine_over_gloo():
    out = spawn(chunk_a2a_case)
    world, E_loc, C, n = 2, 3, 7, 3
    sizes, starts = O.partition_sizes(C, n), O.chunk_starts(C, n)
    for d in range(world):
        full, rings, back, src = out[d]
        for el in range(E_loc):
            e = d * E_loc + el
            for i in range(n):
                c_i, s_i = sizes[i], starts[i]
                # oracle all-to-all: chunk i of expert (d, el) = its slots [s_i, s_i+c_i) from every source
                expect = np.concatenate([out[s][3][e, s_i:s_i + c_i] for s in range(world)])
                np.testing.assert_array_equal(full[el, world * s_i: world * (s_i + c_i)], expect)
                np.testing.assert_array_equal(rings[i][el], expect)
        np.testing.assert_array_equal(back, src)  # combine inverts dispatch


def test_block_plan_single_rank_is_identity_layout():
    # N = 1, full buffer: block (0, el) of chunk i maps slot rows onto themselves
    peers, soff, roff = block_plan(_lib.A2A_DISPATCH, 1, 4, 3, 10, 9, 3, 9, 3)
    assert peers == [0] * 4 and soff == roff == [(el * 9 + 3) * 10 for el in range(4)]


def decisions_case(rank, world):
    from paper_2506_22175_b200.calibrate import _max_over_ranks
    from paper_2506_22175_b200.granularity import AdaptiveController, TrialBudget
    from paper_2506_22175_b200.spec import NO_REUSE, ModelSpec

    rng = np.random.default_rng(100 + rank)  # rank-local measurement noise

    def adapter(spec, hw, strategy, tokens, n):
        best = 2 if tokens < 8192 else 4
        return _max_over_ranks(abs(n - best) + 0.3 * rng.random() + n * 1e-6)

    ctrl = AdaptiveController(ModelSpec(64, 256, 8, world), None, NO_REUSE,
                              TrialBudget(candidates=(1, 2, 4, 8), adapter=adapter))
    work = [1024 * (1 + (i * 7) % 24) for i in range(40)]
    return [ctrl.adaptive_granularity(b) for b in work], ctrl.index.ranges


def test_algorithm1_decisions_are_rank_symmetric():
    out = spawn(decisions_case)
    assert out[0] == out[1]


def gate_grad_case(rank, world):
    g = torch.full((4, 8), float(rank + 1))
    dist.all_reduce(g)
    return g.numpy()


def test_gate_gradient_all_reduce_sums_ranks():
    out = spawn(gate_grad_case)
    np.testing.assert_array_equal(out[0], np.full((4, 8), 3.0))
    np.testing.assert_array_equal(out[0], out[1])


def test_oracle_multi_rank_layout_matches_block_plan_semantics():
    """The oracle's expert input (rows ordered (source, slot)) is what the plan builds."""
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal((40, 8)) for _ in range(2)]
    res = O.moe_layer(xs, rng.standard_normal((4, 8)), [rng.standard_normal((2, 6, 8))] * 2,
                      [rng.standard_normal((2, 8, 6))] * 2, k=2, capacity_factor=1.0, n_chunks=2)
    assert len(res.y) == 2 and res.y[0].shape == (40, 8)
