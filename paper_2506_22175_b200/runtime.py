"""Executes a schedule DAG (schedule.build_schedule) on three CUDA streams.

This is where the reference's model becomes the machine: every OpNode is
issued on its stream ("compute", "collective", "copy"; core.py:24-28) in
the DAG's per-stream FIFO issue order (schedule.py:180-195, 382-386);
every dependency on another stream becomes a cudaStreamWaitEvent on that
op's end event; every SlotSpec acquisition takes the next buffer of its
pool's ring (capacity 2/1 with reuse, n without, schedule.py:363-376) and
first waits for the end events of the ops that released the buffer's
previous occupant — the "slot overwritten while still needed" hazard that
replay_validate (trace.py) re-checks on the measured timeline.

Host issue order: the executor merges the three stream orders into one
host order in which every op comes after its dependencies and after the
releasers of the slot it recycles, so each event it waits on has already
been recorded (waiting on an unrecorded event would silently not wait).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import torch

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
    buffers: list[torch.Tensor] = field(default_factory=list)
    alias: Callable[[int], torch.Tensor] | None = None
    # runtime state
    seq: int = 0
    occupant_releases: dict[int, list[str]] = field(default_factory=dict)
    by_partition: dict[int, torch.Tensor] = field(default_factory=dict)

    def reset_ring(self) -> None:
        self.seq = 0
        self.occupant_releases.clear()


class PipelineExecutor:
    """Issue a ScheduleDag's ops onto CUDA streams with event-guarded slots."""

    def __init__(self, dag: ScheduleDag, streams: dict[str, torch.cuda.Stream],
                 impl: Callable[[str, "PipelineExecutor"], None], pools: dict[str, Pool],
                 record_times: bool = False) -> None:
        self.dag = dag
        self.streams = streams
        self.impl = impl
        self.pools = pools
        self.record_times = record_times
        self.end_events: dict[str, torch.cuda.Event] = {}
        self.start_events: dict[str, torch.cuda.Event] = {}
        self._acq: dict[str, list[tuple[int, object]]] = {}
        for idx, slot in enumerate(dag.slots):
            if slot.acquire is not None:
                self._acq.setdefault(slot.acquire, []).append((idx, slot))
        self.host_order: list[str] = []

    # ------------------------------------------------------------- helpers
    def buffer(self, pool: str, partition: int) -> torch.Tensor:
        """The buffer `pool` holds for `partition` (set at its acquisition)."""
        p = self.pools[pool]
        if p.alias is not None:
            return p.alias(partition)
        try:
            return p.by_partition[partition]
        except KeyError:
            raise ScheduleError(f"pool {pool} holds no buffer for partition {partition}") from None

    def stream_of(self, op_id: str) -> torch.cuda.Stream:
        return self.streams[self.dag.ops[op_id].stream]

    # ---------------------------------------------------------------- plan
    def _plan(self) -> list[tuple[str, list[str], list[tuple[str, int]]]]:
        """Host order with, per op, the release ops to wait for and its slot picks."""
        dag = self.dag
        heads = {s: 0 for s in STREAMS}
        issued: set[str] = set()
        seq = {name: p.seq for name, p in self.pools.items()}
        occupants = {name: dict(p.occupant_releases) for name, p in self.pools.items()}
        plan = []
        total = len(dag.ops)
        while len(issued) < total:
            progressed = False
            for s in STREAMS:
                order = dag.issue_order.get(s, ())
                if heads[s] >= len(order):
                    continue
                op_id = order[heads[s]]
                if any(d not in issued for d in dag.ops[op_id].deps):
                    continue
                waits, picks, ok = [], [], True
                local = {}
                for _, slot in self._acq.get(op_id, ()):
                    p = self.pools.get(slot.pool)
                    if p is None or p.alias is not None:  # full-size / aliased: no ring
                        continue
                    k = local.get(slot.pool, 0)
                    local[slot.pool] = k + 1
                    b = (seq[slot.pool] + k) % p.capacity
                    prev = occupants[slot.pool].get(b)
                    if prev is not None:
                        if not prev:  # held to the end: the ring cannot wrap onto it
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
                picks = [(pool, b) for pool, b, _ in picks]
                plan.append((op_id, waits, picks))
                issued.add(op_id)
                heads[s] += 1
                progressed = True
            if not progressed:
                heads_desc = {s: dag.issue_order[s][heads[s]] for s in STREAMS
                              if heads[s] < len(dag.issue_order.get(s, ()))}
                raise ScheduleError(f"host issue deadlock at stream heads {heads_desc}")
        for name, p in self.pools.items():
            p.seq = seq[name]
            p.occupant_releases = occupants[name]
        return plan

    # ----------------------------------------------------------------- run
    def run(self, after: torch.cuda.Event | None = None) -> None:
        """Issue every op. `after`: event all streams wait for before their first op."""
        plan = self._plan()
        first_on: set[str] = set()
        for op_id, release_waits, picks in plan:
            node = self.dag.ops[op_id]
            stream = self.streams[node.stream]
            if after is not None and node.stream not in first_on:
                stream.wait_event(after)
                first_on.add(node.stream)
            for dep in node.deps:
                if self.dag.ops[dep].stream != node.stream:
                    stream.wait_event(self.end_events[dep])
            for rel in release_waits:
                if self.dag.ops[rel].stream != node.stream:
                    stream.wait_event(self.end_events[rel])
            for pool, b in picks:
                self.pools[pool].by_partition[node.partition] = self.pools[pool].buffers[b]
            with torch.cuda.stream(stream):
                if self.record_times:
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(stream)
                    self.start_events[op_id] = ev
                self.impl(op_id, self)
                end = torch.cuda.Event(enable_timing=self.record_times)
                end.record(stream)
                self.end_events[op_id] = end
            self.host_order.append(op_id)

    def join(self, stream: torch.cuda.Stream) -> None:
        """Make `stream` wait for the last op of every stream."""
        for s in STREAMS:
            order = self.dag.issue_order.get(s, ())
            if order and self.streams[s] is not stream:
                stream.wait_event(self.end_events[order[-1]])

    def times(self, origin: torch.cuda.Event) -> dict[str, tuple[float, float]]:
        """Measured (start, end) seconds of every op relative to `origin` (synchronises)."""
        if not self.record_times:
            raise RuntimeError("executor was not recording times")
        torch.cuda.synchronize()
        return {o: (origin.elapsed_time(self.start_events[o]) * 1e-3,
                    origin.elapsed_time(self.end_events[o]) * 1e-3) for o in self.dag.ops}
