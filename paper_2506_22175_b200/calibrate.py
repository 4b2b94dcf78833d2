"""On-device measurement: the HardwareProfile and the Algorithm-1 adapter.

The reference leaves both seams pluggable and fills them with a simulator
and a synthetic profile (autotune.py:37-51, cli.py:55-68).  Here they are
measured on the B200 the layer runs on:

  measure_profile(layer)   HardwareProfile (core.py:183-243): w_comp from a
                           timed tcgen05 grouped GEMM (element-ops/s in the
                           reference's unit b*H*M), w_comm from a timed
                           chunk exchange of the layer's communicator
                           (peer-memory pull or NCCL; N > 1; at N == 1 the collective
                           stream carries no bytes), w_mem from a timed
                           pinned D2H copy, the comp/mem interference
                           factors from running GEMM and copy concurrently,
                           and the comp/comm ones (mu_comp, sigma_comm) from
                           running the exchange copy kernel beside the GEMM.
  GpuMeasurementAdapter    MeasurementAdapter (autotune.py:33-34): CUDA-event
                           time of one real forward+backward of the layer at
                           (routed tokens, n, strategy) — a CUDA-graph replay
                           of the step on one rank, the eager step (max over
                           EP ranks, so every rank takes the same decision)
                           otherwise.
"""

from __future__ import annotations

import ctypes
import statistics

import torch
import torch.distributed as dist

from . import _lib, ops
from .spec import HardwareProfile, SlowdownTable


def _time(fn, reps: int = 3, warmup: int = 1, stream=None, min_ms: float = 0.0) -> float:
    """Median seconds of fn() measured with CUDA events on `stream`.  min_ms > 0: at least that much
    device time of warm-up and of timed calls (short steps get more repetitions, so a trial's median is
    not one or two launches' jitter)."""
    stream = stream or torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    if min_ms > 0:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        one = max(a.elapsed_time(b), 1e-3)
        for _ in range(int(min_ms / 2 / one)):  # warm-up to the steady (power-limited) clock
            fn()
        reps = max(reps, min(64, int(min_ms / one) + 1))
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        out.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(out)


def _max_over_ranks(value: float, group=None) -> float:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        t = torch.tensor([value], dtype=torch.float64,
                         device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return float(t.item())
    return value


def measure_profile(layer, micro_batch: int = 4096, tokens: int | None = None) -> HardwareProfile:
    """Measure w_comp / w_comm / w_mem, compute saturation and comp-vs-copy interference for `layer`.

    w_comp and compute_saturation (the reference's b_sat: rate = w_comp *
    min(1, b / b_sat), core.py:229-231) come from the expert GEMMs of one
    chunk (fc1 + fc2, 2 work units of b*H*M) timed at the full routed
    micro-batch of `tokens` per rank and at 1/2 ... 1/16 of it, so the
    small-chunk tile inefficiency at large n is in the profile.
    """
    dev = layer.w1.device
    dt = layer.w1.dtype
    M, H = layer.d_model, layer.d_hidden
    e_loc = layer.w1.shape[0]
    b_full = micro_batch if tokens is None else layer.num_experts * layer.capacity(tokens)
    rates = {}
    for div in (1, 2, 4, 8, 16):
        r_e = max(1, b_full // div // max(e_loc, 1))  # rows per local expert in one chunk
        b = r_e * e_loc
        a_ = torch.randn(e_loc, r_e, M, device=dev).to(dt)
        h_ = torch.empty(e_loc, r_e, H, device=dev, dtype=dt)
        o_ = torch.empty(e_loc, r_e, M, device=dev, dtype=dt)

        def chunk_gemms(a_=a_, h_=h_, o_=o_):
            ops.gemm(a_, layer.w1, h_, epilogue=_lib.EPI_RELU)
            ops.gemm(h_, layer.w2, o_)

        rates[b] = 2.0 * b * H * M / _time(chunk_gemms)
    w_comp = max(rates.values())
    below = [b * w_comp / r for b, r in rates.items() if r < 0.9 * w_comp]
    b_sat = int(round(statistics.median(below))) if below else 1
    rows = max(1, b_full // max(e_loc, 1))
    a = torch.randn(e_loc, rows, M, device=dev).to(dt)
    c = torch.empty(e_loc, rows, H, device=dev, dtype=dt)
    gemm = lambda: ops.gemm(a, layer.w1, c, epilogue=_lib.EPI_RELU)
    t_gemm = _time(gemm)

    n_host = e_loc * rows * M
    host = torch.empty(n_host, dtype=dt, pin_memory=True)
    src = a.reshape(-1)
    copy_stream = layer._stream("copy")
    copy = lambda: ops.copy_async(host, src, stream=copy_stream)
    t_copy = _time(copy, stream=copy_stream)
    w_mem = n_host / t_copy

    # concurrent GEMM + copy: slowdown of each against its solo time
    start = torch.cuda.Event(enable_timing=True)
    ends = {}

    def both():
        start.record(torch.cuda.current_stream())
        copy_stream.wait_event(start)
        copy()
        gemm()
        e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e1.record(torch.cuda.current_stream())
        e2.record(copy_stream)
        ends["g"], ends["c"] = e1, e2

    both()
    torch.cuda.synchronize()
    both()
    torch.cuda.synchronize()
    tg = start.elapsed_time(ends["g"]) * 1e-3
    tc = start.elapsed_time(ends["c"]) * 1e-3
    sigma_mem = min(1.0, t_gemm / tg) if tg > 0 else 1.0
    eta_comp = min(1.0, t_copy / tc) if tc > 0 else 1.0

    # comm vs comp: the exchange copy kernel (csrc/p2p.cu, the kernel every chunk exchange runs)
    # beside the GEMM.  N > 1 (peer memory): a chunk's pull from every peer's window over NVLink;
    # N == 1: the same kernel on a chunk's worth of local rows (SM co-residency, no NVLink).
    mu_comp, sigma_comm = _comm_interference(layer, gemm, t_gemm, rows, e_loc, M, dt)

    comm = layer.comm
    if comm.nranks > 1 and getattr(comm, "kind", None) == "p2p":
        c_i = max(1, rows // comm.nranks)
        t_a2a, elems = comm.measure_a2a(e_loc, c_i, M, dt)
        w_comm = elems / _max_over_ranks(t_a2a, layer.group)
    elif comm.nranks > 1:
        c_i = max(1, rows // comm.nranks)
        sbuf = torch.randn(comm.nranks * e_loc * c_i * M, device=dev).to(dt)
        rbuf = torch.empty_like(sbuf)
        from .comm import block_plan
        plan = block_plan(_lib.A2A_DISPATCH, comm.nranks, e_loc, c_i, M, c_i, 0, comm.nranks * c_i, 0)
        a2a = lambda: comm.a2a(_lib.A2A_DISPATCH, sbuf, rbuf, plan, c_i * M)
        t_a2a = _max_over_ranks(_time(a2a), layer.group)
        w_comm = sbuf.numel() / t_a2a
    else:
        # N == 1: dispatch/combine are identities (no bytes on the collective stream)
        w_comm = 1e30
    w_comp = _max_over_ranks(1.0 / w_comp, layer.group) ** -1
    b_sat = int(_max_over_ranks(float(b_sat), layer.group))
    w_mem = _max_over_ranks(1.0 / w_mem, layer.group) ** -1
    mu_comp = 1.0 / _max_over_ranks(1.0 / max(mu_comp, 1e-3), layer.group)
    sigma_comm = 1.0 / _max_over_ranks(1.0 / max(sigma_comm, 1e-3), layer.group)
    table = SlowdownTable.from_factors(sigma_mem=max(sigma_mem, 1e-3), eta_comp=max(eta_comp, 1e-3),
                                       mu_comp=mu_comp, sigma_comm=sigma_comm)
    return HardwareProfile(w_comp, w_comm, w_mem, table, launch_overhead=5e-6, compute_saturation=max(1, b_sat))


def _comm_interference(layer, gemm, t_gemm: float, rows: int, e_loc: int, M: int, dt) -> tuple[float, float]:
    """(mu_comp, sigma_comm): rate factors of the exchange copy kernel while the GEMM runs and of the
    GEMM while the copy kernel runs (each solo time over its time when both start together)."""
    from .comm import PeerComm, lower_plan
    comm = layer.comm
    dev = layer.w1.device
    N = comm.nranks
    c_i = max(1, rows // max(N, 1))
    esz = torch.empty((), dtype=dt).element_size()
    xs = layer._stream("collective")
    counter = torch.zeros(1, device=dev, dtype=torch.int32)
    keep = []
    if N > 1 and isinstance(comm, PeerComm):
        from .comm import WindowLayout, Window, pull_plan
        L = WindowLayout(N, N * e_loc, c_i, M, esz, 1, 4)
        win = Window(comm, L.total)
        dst = torch.empty(e_loc * N * c_i * M, device=dev, dtype=dt)
        plan = pull_plan(L, comm.rank, e_loc, c_i, c_i, 0, "t_i", None, ("loc", "x", 0), N * c_i, 0)
        lowered = lower_plan(plan, win.bases, {"x": dst.data_ptr()}, counter.data_ptr())
        keep += [win, dst]
    elif N == 1:
        src = torch.empty(e_loc * c_i * M, device=dev, dtype=dt)
        dst = torch.empty_like(src)
        rb = M * esz
        plan = {"wait": [], "copy": [(("loc", "d", 0), ("loc", "s", 0), c_i * rb, c_i * rb, c_i * rb, e_loc)],
                "signal": [], "arrive": [], "reset": []}
        lowered = lower_plan(plan, [], {"d": dst.data_ptr(), "s": src.data_ptr()}, counter.data_ptr())
        keep += [src, dst]
    else:  # NCCL baseline: its kernels do not co-reside with the persistent GEMM
        return 1.0, 1.0
    one = ctypes.c_uint32(1)
    exch = lambda: _lib.call("mpm_p2p_run", ctypes.byref(lowered), one, ctypes.c_void_p(xs.cuda_stream))
    if N > 1:
        dist.barrier(group=layer.group)
    t_x = _time(exch, stream=xs)
    start = torch.cuda.Event(enable_timing=True)
    ends = {}

    def both():
        start.record(torch.cuda.current_stream())
        xs.wait_event(start)
        exch()
        gemm()
        e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e1.record(torch.cuda.current_stream())
        e2.record(xs)
        ends["g"], ends["x"] = e1, e2

    for _ in range(2):
        if N > 1:
            dist.barrier(group=layer.group)
        both()
        torch.cuda.synchronize()
    tg = start.elapsed_time(ends["g"]) * 1e-3
    tx = start.elapsed_time(ends["x"]) * 1e-3
    if keep and N > 1:
        keep[0].close()
    sigma_comm = min(1.0, t_gemm / tg) if tg > 0 else 1.0
    mu_comp = min(1.0, t_x / tx) if tx > 0 else 1.0
    return mu_comp, sigma_comm


class GpuMeasurementAdapter:
    """Algorithm-1 measurement: timed forward+backward of `layer` at (tokens, n).

    The step is a CUDA-graph replay (layer.StepGraph: single rank, or expert parallel over peer
    memory, whose exchanges replay unchanged), so small-batch trials measure device time rather
    than host launch cost; the NCCL baseline times the eager step.  Expert-parallel trials take
    the max over ranks, so every rank makes the same decision."""

    # warm-up replays bring every candidate to the same steady (power-limited) clock before its timed
    # replays: a single replay right after graph capture runs at the idle boost clock and would favour
    # whichever candidate happens to follow an idle gap
    def __init__(self, layer, reps: int = 4, warmup: int = 3, seed: int = 1234, graphs: bool | None = None,
                 min_ms: float = 20.0) -> None:
        self.layer = layer
        self.reps, self.warmup, self.seed, self.min_ms = reps, warmup, seed, min_ms
        if graphs is None:
            graphs = layer.comm.nranks == 1 or getattr(layer.comm, "kind", None) == "p2p"
        self.graphs = graphs
        self.calls = 0
        self.log: list[tuple[int, int, str, float]] = []  # (tokens, partitions, strategy, seconds) per trial
        # every candidate of a search is timed in alternation with the n = 1 step (the anchor) and
        # reported as anchor time x the median candidate / anchor ratio, so the power-limited clock
        # drifting between consecutive candidates does not pick a slower n
        self._anchor = None  # (tokens, strategy name, StepGraph, seconds)

    def __call__(self, spec, hw, strategy, tokens: int, partitions: int) -> float:
        lay = self.layer
        T = -(-tokens // lay.top_k)
        gen = torch.Generator(device=lay.w1.device).manual_seed(self.seed)
        x = torch.randn(T, lay.d_model, device=lay.w1.device, generator=gen).to(lay.w1.dtype)
        dy = torch.randn(T, lay.d_model, device=lay.w1.device, generator=gen).to(lay.w1.dtype)
        self.calls += 1
        if self.graphs:
            t = self._anchored(T, x, dy, strategy, partitions)
            self.log.append((tokens, partitions, getattr(strategy, "name", str(strategy)), t))
            return t
        # eager (the NCCL baseline backend, which cannot be captured): fixed repetitions on every rank

        def run():
            with torch.no_grad():
                lay.run_step(x, dy, partitions, strategy)

        t = _max_over_ranks(_time(run, reps=self.reps, warmup=self.warmup,
                                  min_ms=self.min_ms if lay.comm.nranks == 1 else 0.0), lay.group)
        self.log.append((tokens, partitions, getattr(strategy, "name", str(strategy)), t))
        return t

    def _anchored(self, T: int, x, dy, strategy, partitions: int, rounds: int = 4) -> float:
        """Candidate time = anchor (n = 1) time x the median of candidate / anchor over alternating rounds.
        Expert parallel: the graphs' replays are lock-step collectives, so every rank replays a fixed
        number of times (no time-based repetitions) and the result is the max over ranks."""
        lay = self.layer
        single = lay.comm.nranks == 1
        min_ms = self.min_ms if single else 0.0
        key = (T, getattr(strategy, "name", str(strategy)))
        if self._anchor is None or self._anchor[:2] != key:
            self.close()
            ref = lay.step_graph(T, 1, strategy)
            ref.x.copy_(x)
            ref.dy.copy_(dy)
            if not single:
                dist.barrier(group=lay.group)
            t0 = _max_over_ranks(_time(ref.graph.replay, reps=self.reps, warmup=self.warmup, min_ms=min_ms), lay.group)
            self._anchor = (*key, ref, t0)
        ref, t_ref = self._anchor[2], self._anchor[3]
        if partitions == 1:
            return t_ref
        sg = lay.step_graph(T, partitions, strategy)
        sg.x.copy_(x)
        sg.dy.copy_(dy)
        if not single:
            dist.barrier(group=lay.group)
        ratios = []
        for _ in range(rounds):  # alternate: both see the same clock within a round
            tc = _time(sg.graph.replay, reps=self.reps, warmup=self.warmup, min_ms=min_ms / rounds)
            tr = _time(ref.graph.replay, reps=self.reps, warmup=1, min_ms=min_ms / rounds)
            ratios.append(tc / tr)
        sg.close()
        return _max_over_ranks(t_ref * statistics.median(ratios), lay.group)

    def close(self) -> None:
        """Release the anchor step graph (its private arena)."""
        if self._anchor is not None:
            self._anchor[2].close()
            self._anchor = None
