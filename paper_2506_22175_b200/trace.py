"""Measured pipeline traces: validation, memory accounting, export.

The runtime (runtime.PipelineExecutor) brackets every schedule op with CUDA
events on the op's own stream (after its cross-stream waits), so a measured
trace has the same shape as the reference simulator's ScheduleTrace
(pipesim/engine.py:46-111) and is checked and exported by the reference's
rules:

  replay_validate     engine.py:427-487  per-stream FIFO / no overlap, deps
                                         respected, pool capacity never
                                         exceeded (no ring slot reused early)
  memory_components   engine.py:329-400  allocated-capacity convention
  to_jsonl / to_trace_event / write_trace   export.py:16-72 (integer-us,
                                         half-up; Chrome trace-event JSON)

plus the metric the reference only implies: exposed (non-overlapped)
all-to-all time = |collective busy \\ compute busy|.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

from .memory import mem_model_states
from .schedule import ACTIVATION, GRADIENT, ScheduleDag
from .spec import COLLECTIVE_STREAM, COMPUTE_STREAM, STREAMS


class TraceInvariantError(AssertionError):
    """A trace violates a schedule invariant."""


@dataclass(frozen=True)
class TraceEvent:
    op_id: str
    kind: str
    partition: int
    stream: str
    start: float   # seconds from the trace origin
    end: float
    segments: tuple[tuple[float, float, float], ...] = ()

    @property
    def duration(self) -> float:
        return self.end - self.start


@dataclass(frozen=True)
class SlotInterval:
    pool: str
    acquired: float
    released: float | None


@dataclass(frozen=True)
class ScheduleTrace:
    dag: ScheduleDag
    events: tuple[TraceEvent, ...]
    slot_intervals: tuple[SlotInterval, ...]
    # op_id -> lane (> 0) for ops executed on an extra physical stream of their
    # logical stream (runtime.PipelineExecutor lanes); FIFO holds within a lane
    lanes: dict = field(default_factory=dict)

    @property
    def makespan(self) -> float:
        return max((e.end for e in self.events), default=0.0)

    def busy_time(self, stream: str) -> float:
        """Time the stream is busy: the union of its ops' intervals (the sum, for FIFO traces)."""
        return sum(b - a for a, b in _union([(e.start, e.end) for e in self.events if e.stream == stream]))

    def by_op(self) -> dict[str, TraceEvent]:
        return {e.op_id: e for e in self.events}

    def bottleneck_stream(self) -> str:
        return max(STREAMS, key=self.busy_time)


def trace_from_times(dag: ScheduleDag, times: dict[str, tuple[float, float]],
                     lanes: dict | None = None) -> ScheduleTrace:
    """Build a trace from measured {op_id: (start, end)} and derive slot intervals."""
    events = tuple(sorted(
        (TraceEvent(o, dag.ops[o].kind, dag.ops[o].partition, dag.ops[o].stream, s, e)
         for o, (s, e) in times.items()),
        key=lambda ev: (ev.start, ev.stream, ev.op_id)))
    intervals = []
    for slot in dag.slots:
        acq = 0.0 if slot.acquire is None else times[slot.acquire][0]
        rel = max((times[r][1] for r in slot.releases), default=None) if slot.releases else None
        intervals.append(SlotInterval(slot.pool, acq, rel))
    return ScheduleTrace(dag, events, tuple(intervals), dict(lanes or {}))


def _union(intervals: list[tuple[float, float]]) -> list[tuple[float, float]]:
    out: list[list[float]] = []
    for a, b in sorted(intervals):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return [(a, b) for a, b in out]


def exposed_time(trace: ScheduleTrace, stream: str = COLLECTIVE_STREAM,
                 against: str = COMPUTE_STREAM) -> float:
    """Length of `stream`'s busy set not covered by `against`'s busy set."""
    busy = _union([(e.start, e.end) for e in trace.events if e.stream == stream])
    cover = _union([(e.start, e.end) for e in trace.events if e.stream == against])
    total, j = 0.0, 0
    for a, b in busy:
        covered = 0.0
        for c, d in cover:
            lo, hi = max(a, c), min(b, d)
            if hi > lo:
                covered += hi - lo
        total += (b - a) - covered
    return total


def exposed_a2a_fraction(trace: ScheduleTrace) -> float:
    span = trace.makespan - min((e.start for e in trace.events), default=0.0)
    return exposed_time(trace) / span if span > 0 else 0.0


@dataclass(frozen=True)
class MemoryComponents:
    model_states: int
    activations: int
    buffers: int
    host: int
    element_bytes: int

    @property
    def total(self) -> int:
        return self.model_states + self.activations + self.buffers

    def to_dict(self) -> dict:
        return {"model_states_elements": self.model_states, "activations_elements": self.activations,
                "buffers_elements": self.buffers, "total_elements": self.total,
                "host_elements": self.host, "total_bytes": self.total * self.element_bytes,
                "host_bytes": self.host * self.element_bytes}


def _liveness_peak(trace: ScheduleTrace, category: str) -> int:
    pools = trace.dag.pools
    end = trace.makespan
    edges = []
    for iv in trace.slot_intervals:
        p = pools[iv.pool]
        if p.category == category:
            edges.append((iv.acquired, 1, p.slot_elements))
            edges.append((end if iv.released is None else iv.released, 0, -p.slot_elements))
    level = peak = 0
    for _, _, d in sorted(edges, key=lambda x: (x[0], x[1])):
        level += d
        peak = max(peak, level)
    return peak


def memory_components(trace: ScheduleTrace) -> MemoryComponents:
    """Peak device elements: capacity sums, except the n=1 backward (liveness)."""
    dag = trace.dag
    cap = lambda cat: sum(p.capacity * p.slot_elements for p in dag.pools.values() if p.category == cat)
    if not dag.includes_backward:
        buf = 0
    elif dag.batch.partitions == 1:
        buf = _liveness_peak(trace, GRADIENT)
    else:
        buf = cap(GRADIENT)
    return MemoryComponents(mem_model_states(dag.spec), cap(ACTIVATION), buf,
                            sum(h.elements for h in dag.host_slices), dag.spec.element_bytes)


def peak_memory(trace: ScheduleTrace, spec=None, batch=None, strategy=None, reuse_enabled=None) -> int:
    dag = trace.dag
    if spec is not None and spec != dag.spec:
        raise ValueError("trace was produced for a different model spec")
    if batch is not None and batch != dag.batch:
        raise ValueError("trace was produced for a different batch spec")
    if strategy is not None and strategy.name != dag.strategy.name:
        raise ValueError("trace was produced for a different strategy")
    if reuse_enabled is not None and reuse_enabled != dag.reuse_enabled:
        raise ValueError("trace reuse flag mismatch")
    return memory_components(trace).total


def replay_validate(trace: ScheduleTrace, slack: float = 2e-6) -> None:
    """Schedule invariants on a (measured) trace; `slack` absorbs timer skew."""
    dag = trace.dag
    ev = trace.by_op()
    if set(ev) != set(dag.ops):
        raise TraceInvariantError("trace does not cover the DAG's ops exactly")
    for stream, order in dag.issue_order.items():
        for lane in sorted({trace.lanes.get(o, 0) for o in order}):  # FIFO within each lane
            seq = [ev[o] for o in order if trace.lanes.get(o, 0) == lane]
            for a, b in zip(seq, seq[1:]):
                if b.start + slack < a.end:
                    raise TraceInvariantError(f"{stream}: {b.op_id} starts before {a.op_id} ends")
                if b.start + slack < a.start:
                    raise TraceInvariantError(f"{stream}: starts out of issue order")
    for op_id, node in dag.ops.items():
        for d in node.deps:
            if ev[op_id].start + slack < ev[d].end:
                raise TraceInvariantError(f"{op_id} started before dependency {d} ended")
        segs = ev[op_id].segments
        if segs:
            worked = sum((b - a) * r for a, b, r in segs)
            if abs(worked - node.work) > 1e-9 * max(abs(node.work), 1.0):
                raise TraceInvariantError(f"{op_id}: integrated work {worked} != {node.work}")
    end = trace.makespan
    edges = []
    for iv in trace.slot_intervals:
        edges.append((iv.acquired, 1, iv.pool))
        edges.append((end if iv.released is None else iv.released - slack, 0, iv.pool))
    level = {p: 0 for p in dag.pools}
    for _, acquire, pool in sorted(edges, key=lambda x: (x[0], x[1])):
        level[pool] += 1 if acquire else -1
        if level[pool] > dag.pools[pool].capacity:
            raise TraceInvariantError(f"pool {pool} exceeded capacity {dag.pools[pool].capacity}")


# ---------------------------------------------------------------- export
def us(seconds: float) -> int:
    """Integer microseconds, half-up."""
    return int(math.floor(seconds * 1e6 + 0.5))


def event_rows(trace: ScheduleTrace) -> list[dict]:
    return [{"op": e.op_id, "kind": e.kind, "partition": e.partition, "stream": e.stream,
             "start_us": us(e.start), "end_us": us(e.end)} for e in trace.events]


def to_jsonl(trace: ScheduleTrace) -> str:
    rows = [json.dumps(r, sort_keys=True) for r in event_rows(trace)]
    return "".join(r + "\n" for r in rows)


def to_trace_event(trace: ScheduleTrace) -> dict:
    tid = {s: i for i, s in enumerate(STREAMS)}
    out = []
    for e in trace.events:
        t0 = us(e.start)
        out.append({"name": e.op_id, "cat": e.kind, "ph": "X", "ts": t0, "dur": us(e.end) - t0,
                    "pid": 0, "tid": tid[e.stream], "args": {"partition": e.partition, "stream": e.stream}})
    return {"traceEvents": out, "displayTimeUnit": "ms"}


def write_trace(trace: ScheduleTrace, path: str, fmt: str = "jsonl") -> None:
    if fmt == "jsonl":
        text = to_jsonl(trace)
    elif fmt == "trace-event":
        text = json.dumps(to_trace_event(trace), sort_keys=True)
    else:
        raise ValueError(f"unknown trace format {fmt!r}; use jsonl or trace-event")
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(text)
