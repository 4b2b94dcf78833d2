"""Host-side issue planning of runtime.PipelineExecutor (no GPU needed).

The plan must (a) keep every stream's FIFO order, (b) put every op after its
dependencies and after the ops releasing the ring slot it recycles, and
(c) never hand one ring buffer to two live occupants.  These are the
reference's schedule invariants (pipesim/engine.py:427-487) checked on the
plan the CUDA streams will execute.
"""

import itertools

import pytest
import torch

from paper_2506_22175_b200.runtime import Pool, plan_dag
from paper_2506_22175_b200.schedule import BACKWARD, BOTH, FORWARD, build_schedule
from paper_2506_22175_b200.spec import NO_REUSE, STRATEGIES, BatchSpec, ModelSpec

SPEC = ModelSpec(16, 64, 8, 2)


def make_pools(dag, alias_io: bool):
    pools = {}
    for name, p in dag.pools.items():
        if name in ("t_i", "t_o", "g_o", "g_i"):
            continue
        if alias_io and name in ("t_di", "t_do", "g_do", "g_di"):
            pools[name] = Pool(name, 1, alias=lambda i: torch.empty(1))
        else:
            pools[name] = Pool(name, p.capacity, [torch.empty(1) for _ in range(p.capacity)])
    return pools


def check_plan(dag, plan):
    pos = {op: i for i, (op, _, _) in enumerate(plan)}
    assert set(pos) == set(dag.ops)
    for s, order in dag.issue_order.items():
        assert [p for p in pos if dag.ops[p].stream == s] == sorted(order, key=pos.get)
        assert [pos[o] for o in order] == sorted(pos[o] for o in order)
    for op, waits, picks in plan:
        for d in dag.ops[op].deps:
            assert pos[d] < pos[op]
        for w in waits:
            assert pos[w] < pos[op]
    # ring occupancy: a buffer is re-acquired only after all releasers of its previous occupant
    owner = {}
    acq = {s.acquire: [] for s in dag.slots}
    for s in dag.slots:
        acq[s.acquire].append(s)
    for op, waits, picks in plan:
        slots = [s for s in acq.get(op, []) if (s.pool, None) not in owner or True]
        for (pool, b) in picks:
            prev = owner.get((pool, b))
            if prev is not None:
                assert prev, "wrapped onto a held slot"
                assert set(prev) <= set(waits) | {o for o, _, _ in plan[:pos[op]]}
            spec = next(s for s in slots if s.pool == pool)
            owner[(pool, b)] = spec.releases


@pytest.mark.parametrize("name,n,direction,alias", list(itertools.product(
    ["none", "s1", "s2", "s3", "s4"], [1, 2, 3, 4, 8], [FORWARD, BACKWARD, BOTH], [False, True])))
def test_plan_respects_schedule(name, n, direction, alias):
    strategy = STRATEGIES[name]
    reuse = strategy.saves_memory and n >= 2
    dag = build_schedule(SPEC, BatchSpec(64 * n, n), strategy if reuse else NO_REUSE, reuse, direction)
    plan = plan_dag(dag, make_pools(dag, alias))
    check_plan(dag, plan)


def test_reuse_plan_waits_for_offload_before_overwrite():
    """S1 forward: chunk i+1's T_M slot (capacity 1) must wait for Dm_i (copy stream)."""
    dag = build_schedule(SPEC, BatchSpec(256, 4), STRATEGIES["s1"], True, FORWARD)
    plan = {op: waits for op, waits, _ in plan_dag(dag, make_pools(dag, False))}
    for i in range(1, 4):
        assert f"Dm{i - 1}" in plan[f"C{i}"]
        assert f"Ddi{i - 2}" in plan[f"S{i}"] if i >= 2 else True


class _FakeEvent:
    def __init__(self, timing=False):
        self.timing = timing


def test_compute_lanes_turn_same_stream_deps_into_event_waits(monkeypatch):
    """With odd chunks' compute ops on a second lane, every dependency or slot release that
    crosses physical streams becomes an event wait, and each lane keeps its own FIFO."""
    import ctypes

    from paper_2506_22175_b200 import runtime
    monkeypatch.setattr(runtime, "Event", _FakeEvent)
    for direction in (FORWARD, BACKWARD):
        dag = build_schedule(SPEC, BatchSpec(256, 4), NO_REUSE, False, direction)
        pools = make_pools(dag, True)
        streams = {s: ctypes.c_void_p(i + 1) for i, s in enumerate(("compute", "collective", "copy"))}
        lane_b = ctypes.c_void_p(99)
        lanes = {o: lane_b for o, node in dag.ops.items() if node.stream == "compute" and node.partition % 2}
        ex = runtime.PipelineExecutor(dag, pools, lambda op: [lambda: None], streams, lanes=lanes)
        where = {op: st for op, st, _, _ in ex.program}
        waits = {op: w for op, _, w, _ in ex.program}
        for op, node in dag.ops.items():
            assert where[op] is (lane_b if op in lanes else streams[node.stream])
            for d in node.deps:  # a dependency on another physical stream is an event wait
                if where[d] is not where[op]:
                    assert ex.end[d] in waits[op], (op, d)
        first = {}
        for op, st, w, _ in ex.program:  # every physical stream first waits for the step origin
            if id(st) not in first:
                first[id(st)] = op
                assert ex.after in w


def test_trace_fifo_is_checked_per_lane():
    from paper_2506_22175_b200.trace import TraceInvariantError, replay_validate, trace_from_times
    dag = build_schedule(SPEC, BatchSpec(256, 2), NO_REUSE, False, FORWARD)
    # C0 and C1 overlap in time (two lanes), all dependencies respected
    t = {"S0": (0.0, 1.0), "S1": (1.0, 2.0), "C0": (1.0, 5.0), "C1": (2.0, 6.0), "R0": (5.0, 6.0),
         "R1": (6.0, 7.0)}
    t = {o: t[o] for o in dag.ops}
    replay_validate(trace_from_times(dag, t, {"C1": 1}))
    with pytest.raises(TraceInvariantError):
        replay_validate(trace_from_times(dag, t))  # one compute lane: C1 starts before C0 ends


def test_busy_time_is_the_union_of_intervals():
    """With two compute lanes a logical stream can run two ops at once: busy time is the union."""
    from paper_2506_22175_b200.trace import exposed_time, trace_from_times
    dag = build_schedule(SPEC, BatchSpec(256, 2), NO_REUSE, False, FORWARD)
    t = {"S0": (0.0, 1.0), "S1": (1.0, 2.0), "C0": (1.0, 5.0), "C1": (2.0, 6.0), "R0": (5.0, 6.0),
         "R1": (6.0, 7.0)}
    tr = trace_from_times(dag, {o: t[o] for o in dag.ops}, {"C1": 1})
    assert tr.busy_time("compute") == 5.0          # [1, 6), not 4 + 4
    assert tr.busy_time("collective") == 4.0       # [0, 2) + [5, 7)
    assert exposed_time(tr) == 2.0                 # collective busy outside compute: [0, 1) and [6, 7)
