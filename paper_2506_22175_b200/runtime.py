"""Executes a schedule DAG (schedule.build_schedule) on three CUDA streams.

This is where the reference's model becomes the machine: every OpNode is
issued on its stream ("compute", "collective", "copy"; core.py:24-28) in
the DAG's per-stream FIFO issue order (schedule.py:180-195, 382-386);
every dependency on another stream becomes a CUDA event wait on that op's
end event; every SlotSpec acquisition takes the next buffer of its pool's
ring (capacity 2/1 with reuse, n without, schedule.py:363-376) and first
waits for the end events of the ops that released the buffer's previous
occupant — the "slot overwritten while still needed" hazard that
replay_validate (trace.py) re-checks on the measured timeline.

Compilation happens once per step arena: the plan (host issue order, ring
picks, cross-stream waits) and every op's C-ABI calls with their argument
blocks are prebuilt, so issuing an op costs a handful of ctypes calls.

Host issue order: the three stream orders are merged into one host order in
which every op comes after its dependencies and after the releasers of the
slot it recycles, so each event it waits on has already been recorded
(waiting on an unrecorded event would silently not wait).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

from ._lib import Event, stream_wait
from .schedule import ScheduleDag, ScheduleError
from .spec import STREAMS


@dataclass
class Pool:
    """Buffers of one slot pool.

    ring: `capacity` preallocated buffers cycled in acquisition order;
    alias: fn(partition) -> view into a full-size tensor (used at N == 1,
    where dispatch/combine are identities and T_DI / T_DO / g_do / g_di are
    the chunk regions of T_I / T_O / g_o / g_i themselves).
    """

    name: str
    capacity: int
    buffers: list = field(default_factory=list)
    alias: Callable | None = None
    seq: int = 0
    occupant_releases: dict = field(default_factory=dict)
    by_partition: dict = field(default_factory=dict)

    def reset_ring(self) -> None:
        self.seq = 0
        self.occupant_releases.clear()

    def get(self, partition: int):
        if self.alias is not None:
            return self.alias(partition)
        try:
            return self.by_partition[partition]
        except KeyError:
            raise ScheduleError(f"pool {self.name} holds no buffer for partition {partition}") from None


def plan_dag(dag: ScheduleDag, pools: dict[str, Pool]) -> list[tuple[str, list[str], list[tuple[str, int]]]]:
    """(op, release ops to wait for, ring picks) in a valid host issue order."""
    acq: dict[str, list] = {}
    for slot in dag.slots:
        if slot.acquire is not None:
            acq.setdefault(slot.acquire, []).append(slot)
    heads = {s: 0 for s in STREAMS}
    issued: set[str] = set()
    seq = {name: p.seq for name, p in pools.items()}
    occupants = {name: dict(p.occupant_releases) for name, p in pools.items()}
    plan = []
    while len(issued) < len(dag.ops):
        progressed = False
        for s in STREAMS:
            order = dag.issue_order.get(s, ())
            if heads[s] >= len(order):
                continue
            op_id = order[heads[s]]
            if any(d not in issued for d in dag.ops[op_id].deps):
                continue
            waits, picks, ok, local = [], [], True, {}
            for slot in acq.get(op_id, ()):
                p = pools.get(slot.pool)
                if p is None or p.alias is not None:  # full-size / aliased: no ring
                    continue
                k = local.get(slot.pool, 0)
                local[slot.pool] = k + 1
                b = (seq[slot.pool] + k) % p.capacity
                prev = occupants[slot.pool].get(b)
                if prev is not None:
                    if not prev:
                        raise ScheduleError(f"pool {slot.pool} wraps onto a slot held to the end")
                    if any(r not in issued for r in prev):
                        ok = False
                        break
                    waits += prev
                picks.append((slot.pool, b, tuple(slot.releases)))
            if not ok:
                continue
            for pool, b, rel in picks:
                occupants[pool][b] = list(rel)
                seq[pool] += 1
            plan.append((op_id, waits, [(pool, b) for pool, b, _ in picks]))
            issued.add(op_id)
            heads[s] += 1
            progressed = True
        if not progressed:
            stuck = {s: dag.issue_order[s][heads[s]] for s in STREAMS if heads[s] < len(dag.issue_order.get(s, ()))}
            raise ScheduleError(f"host issue deadlock at stream heads {stuck}")
    for name, p in pools.items():
        p.seq = seq[name]
        p.occupant_releases = occupants[name]
    return plan


class PipelineExecutor:
    """A compiled DAG: per op, its stream, cross-stream waits and prebuilt calls.

    `lanes` (op_id -> stream handle) runs chosen ops on an extra physical stream
    of their logical stream (B200: consecutive chunks' expert GEMMs on two compute
    lanes, so one chunk's GEMM fills the SMs the other's last wave leaves idle);
    every dependency or slot release across physical streams becomes an event wait,
    so the DAG's data dependencies hold, and FIFO order holds within each lane."""

    def __init__(self, dag: ScheduleDag, pools: dict[str, Pool], build_calls: Callable[[str], list],
                 streams: dict, timing: bool = False, lanes: dict | None = None) -> None:
        self.dag = dag
        self.pools = pools
        self.streams = streams  # name -> mutable ctypes c_void_p
        self.lanes = dict(lanes or {})
        self.timing = timing
        self.plan = plan_dag(dag, pools)
        self.end: dict[str, Event] = {o: Event(timing) for o in dag.ops}
        self.start: dict[str, Event] = {o: Event(True) for o in dag.ops} if timing else {}
        self.after = Event(timing)
        self.program = []
        # Ops without device work (the all-to-alls at N == 1, offload copies of
        # aliased tensors) are elided: their end event stands for the latest
        # producer they depend on, so dependents never hop streams for them.
        self.proxy: dict[str, Event | None] = {}
        first_on: set[int] = set()
        phys = lambda o: self.lanes.get(o, streams[dag.ops[o].stream])  # noqa: E731
        for op_id, release_waits, picks in self.plan:
            node = dag.ops[op_id]
            for pool, b in picks:
                pools[pool].by_partition[node.partition] = pools[pool].buffers[b]
            calls = build_calls(op_id)
            if not calls:
                producers = [self._event_of(d) for d in node.deps]
                producers = [e for e in producers if e is not None]
                self.proxy[op_id] = producers[-1] if len(producers) == 1 else (None if not producers else False)
                if self.proxy[op_id] is not False:
                    continue
                del self.proxy[op_id]  # several producers: keep a real (empty) op to join them
            waits = []
            st = phys(op_id)
            if id(st) not in first_on:
                waits.append(self.after)
                first_on.add(id(st))
            for other in list(node.deps) + list(release_waits):
                if phys(other) is not st or other in self.proxy:
                    ev = self._event_of(other)
                    if ev is not None and ev not in waits:
                        waits.append(ev)
            self.program.append((op_id, st, waits, calls))
        self.host_order = [p[0] for p in self.plan]

    def _event_of(self, op_id: str):
        """End event standing for op_id (its own, or its elided producer's; None = nothing to wait for)."""
        if op_id in self.proxy:
            return self.proxy[op_id]
        return self.end[op_id]

    def run(self, origin_stream) -> None:
        """Issue every op; all streams first wait for `origin_stream`'s current work."""
        self.after.record(origin_stream)
        for op_id, stream, waits, calls in self.program:
            for ev in waits:
                stream_wait(stream, ev)
            if self.timing:
                self.start[op_id].record(stream)
            for c in calls:
                c()
            self.end[op_id].record(stream)

    def join(self, stream, only=None) -> None:
        """Make `stream` wait for the last issued op of every other stream (or of the
        stream handles in `only`)."""
        last: dict = {}
        for op_id, st, _, _ in self.program:
            if only is None or any(st is o for o in only):
                last[st.value] = op_id
        for value, op_id in last.items():
            if value != stream.value:
                stream_wait(stream, self.end[op_id])

    def times(self) -> dict[str, tuple[float, float]]:
        """Measured (start, end) seconds of every op relative to the run's origin (synchronises).

        Elided ops (no device work) are reported as zero-length at the end of
        the producer they stand for (or at the origin)."""
        if not self.timing:
            raise RuntimeError("executor was not built with timing")
        out = {}
        for o in self.dag.ops:
            if o not in self.proxy:
                out[o] = (self.after.elapsed_ms(self.start[o]) * 1e-3, self.after.elapsed_ms(self.end[o]) * 1e-3)
        for stream, order in self.dag.issue_order.items():  # elided ops: FIFO-monotone placeholders
            last = 0.0
            for o in order:
                if o in self.proxy:
                    ev = self.proxy[o]
                    t = max(last, self.after.elapsed_ms(ev) * 1e-3 if ev is not None else 0.0)
                    out[o] = (t, t)
                last = max(last, out[o][1])
        return out
