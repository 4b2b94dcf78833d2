"""MoELayer: the B200-native pipelined expert-parallel MoE layer.

API per the paper (`pmoe.MoELayer(d_model, d_hidden,
top_k, num_experts, pipeline, memory_reuse)`) plus the gate/capacity keys
of the north star and the reference's pipeline vocabulary
(cli.py:86-98: pipeline.n int | "adaptive", candidates,
trials_per_candidate, min_micro_batch, strategy none|s1..s4|auto).

Forward:
  compute stream   gate GEMM -> top-k/softmax -> slot assignment -> permute
                   into the chunk-major send buffer T_I
  schedule DAG     S_i / C_i / R_i (+ Ddi_i, Dm_i) on the collective /
                   compute / copy streams (schedule.build_schedule compiled
                   and issued by runtime.PipelineExecutor)
  compute stream   weighted combine of T_O -> y
Backward mirrors it (combine_bwd -> BS/RC/Hdi/Hm/RE/G2/G1/BR -> gather),
with the gate's own backward (dlogits, dWg, dlogits.Wg — inputs dprob, x,
Wg only) on a side stream under the expert backward, then one all-reduce of the replicated gate's gradient
(data parallel).

Device state lives in a per-step *arena* (the reference's allocated-
capacity convention, engine.py:329-400): full-size T_I / T_O / g_o / g_i,
the slot rings sized by the DAG's pool capacities, routing tensors and the
wgrad accumulators, allocated once per (tokens, n, strategy) and reused by
later steps; every kernel call of the step is prebuilt against it.

The granularity n comes from Algorithm 1 (granularity.AdaptiveController)
with a CUDA-event-timed measurement of this very layer; the reuse strategy
from cost.select_strategy over a HardwareProfile measured on the device
(calibrate.py) when memory_reuse="auto".
"""

from __future__ import annotations

import ctypes
import math
import os
import weakref
from dataclasses import dataclass

import torch
import torch.distributed as dist
from torch import nn

from . import _lib, ops
from ._lib import Call, GemmArgs
from .comm import (
    FLAG_GO_READY,
    FLAG_TI_READY,
    FLAG_XS_FREE,
    WindowLayout,
    block_plan,
    combine_push_plan,
    compact_pull_plan,
    kept_signal_plan,
    lower_plan,
    lower_push,
    make_comm,
    pull_plan,
    push_dispatch_plan,
    push_plan,
    reduce_plan,
    signal_plan,
)
from .runtime import PipelineExecutor, Pool
from .schedule import BACKWARD, FORWARD, build_schedule
from .spec import (
    COLLECTIVE_STREAM,
    COMPUTE_STREAM,
    COPY_STREAM,
    NO_REUSE,
    BatchSpec,
    InvalidPartitioningError,
    ModelSpec,
    RestoreMethod,
    ReuseStrategy,
    balanced_split,
)

_V = ctypes.c_void_p


def _starts(sizes: list[int]) -> list[int]:
    out, acc = [], 0
    for v in sizes:
        out.append(acc)
        acc += v
    return out


@dataclass(frozen=True)
class Chunk:
    """One micro-batch of the pipeline: the routed rows of local experts [e0, e0+ne) in capacity
    slots [s0, s0+cs) from every source rank."""
    e0: int
    ne: int
    s0: int
    cs: int
    part: int  # slot part index (0 .. n_s-1): which mpm_chunk_rows row bounds its valid rows


# Largest expert GEMM of one chunk (256 x 256 pair tiles) that still runs on two compute lanes (_Arena).
LANE_MAX_TILES = 4096

@dataclass(frozen=True)
class Geometry:
    """Per-rank layer geometry and its n-way chunk decomposition.

    The reference splits the routed batch B into n micro-batches (core.py:102-105),
    each a full N-way all-to-all of 1/n of the volume.  Here the split is along local experts first:
    the E_loc local experts form n_e balanced groups (n_e = the largest divisor of n not above E_loc)
    and, when n exceeds that, each group's capacity slots form n_s = n / n_e balanced parts.  Chunk
    i = (group i // n_s, slot part i % n_s).  Every chunk is still a full all-to-all of 1/n of the
    volume, but a chunk's expert GEMMs stream only its own experts' weights (not all E_loc per
    chunk), and with n_s = 1 each expert's weight gradient is produced by exactly one chunk — no
    per-chunk read-modify-write of dW under memory reuse and one rounding of it.
    """
    T: int
    M: int
    H: int
    E: int
    N: int
    rank: int
    k: int
    C: int
    n: int

    @property
    def e_loc(self) -> int:
        return self.E // self.N

    @property
    def n_e(self) -> int:
        return max(d for d in range(1, min(self.n, self.e_loc) + 1) if self.n % d == 0)

    @property
    def n_s(self) -> int:
        return self.n // self.n_e

    @property
    def group_sizes(self) -> list[int]:
        return balanced_split(self.e_loc, self.n_e)

    @property
    def part_sizes(self) -> list[int]:
        return balanced_split(self.C, self.n_s)

    def chunk(self, i: int) -> Chunk:
        gi, si = divmod(i, self.n_s)
        gs, ps = self.group_sizes, self.part_sizes
        return Chunk(_starts(gs)[gi], gs[gi], _starts(ps)[si], ps[si], si)

    def rows(self, i: int) -> int:
        """Rows per local expert in chunk i (all sources)."""
        return self.N * self.chunk(i).cs

    @property
    def max_rows(self) -> int:
        return self.N * max(self.part_sizes)

    @property
    def max_experts(self) -> int:
        return max(self.group_sizes)


def _full_view(buf: torch.Tensor, g: Geometry, i: int, width: int, experts: int, rows_per_slot: int) -> torch.Tensor:
    """Chunk i of an expert-major all-chunk buffer [experts][rows_per_slot*C][width]: experts
    [e0, e0+ne), rows [R*s0, R*(s0+cs)) (R = rows per slot: 1 for the dispatch buffers, N for the
    expert side, where the N sources' cs rows follow each other)."""
    ch = g.chunk(i)
    R = rows_per_slot
    return buf.reshape(experts, R * g.C, width)[ch.e0:ch.e0 + ch.ne, R * ch.s0: R * (ch.s0 + ch.cs), :]


def _ring_view(flat: torch.Tensor, g: Geometry, i: int, width: int) -> torch.Tensor:
    """[ne, N*cs, width] view of a per-chunk ring slot."""
    ch = g.chunk(i)
    R = g.rows(i)
    return flat.reshape(-1)[: ch.ne * R * width].view(ch.ne, R, width)


def _gemm_args(a, b, c, *, a_mn=False, b_mn=False, epilogue=_lib.EPI_NONE, aux=None, valid_rows=None,
               valid_k=None) -> GemmArgs:
    """GemmArgs for C[b] = A[b] . B[b]^T over 3-D views (see ops.gemm); valid_rows / valid_k are
    int32 device vectors (one entry per batch) that bound the rows / K of capacity-padded experts."""
    args = GemmArgs()
    args.dtype = ops.dtype_code(a.dtype)
    args.epilogue = epilogue
    args.batches = a.shape[0]
    args.rows, args.k = (a.shape[2], a.shape[1]) if a_mn else (a.shape[1], a.shape[2])
    args.n = b.shape[2] if b_mn else b.shape[1]
    args.a, args.a_ld, args.a_batch_stride, args.a_mn_major = a.data_ptr(), a.stride(1), a.stride(0), int(a_mn)
    args.b, args.b_ld, args.b_batch_stride, args.b_mn_major = b.data_ptr(), b.stride(1), b.stride(0), int(b_mn)
    args.c, args.c_ld, args.c_batch_stride, args.c_dtype = c.data_ptr(), c.stride(1), c.stride(0), ops.dtype_code(c.dtype)
    if aux is not None:
        args.aux, args.aux_ld, args.aux_batch_stride = aux.data_ptr(), aux.stride(1), aux.stride(0)
    if valid_rows is not None:
        args.valid_rows = valid_rows.data_ptr()
    if valid_k is not None:
        args.valid_k = valid_k.data_ptr()
    return args



class _Arena:
    """Device state + compiled schedule of one in-flight step for one key.

    Layouts (expert-major):
      T_I / T_O / g_o / g_i   [E][C][M]: slot s of expert e at row e*C + s;
                              chunk i = slots [s_i, s_i + c_i) of every expert
      expert side, no reuse   one all-chunk buffer per pool, [E_loc][N*C][W]:
                              chunk i = rows [N*s_i, N*(s_i+c_i)) of every
                              local expert, source-major inside the chunk
                              (at N = 1 these alias T_I / T_O / g_o / g_i)
      expert side, reuse      ring slots of [E_loc][N*c_i][W] (DAG capacities)
    Without reuse every expert's rows of all chunks are contiguous, so each
    weight gradient is one GEMM over K = N*C after the last chunk; with reuse
    the rings are overwritten, so it accumulates per chunk (into the
    parameter-dtype gradient in place, or fp32 accumulators; see
    MoELayer's wgrad_accumulation).
    """

    def __init__(self, layer: "MoELayer", T: int, n: int, strategy: ReuseStrategy, reuse: bool,
                 dtype: torch.dtype, timing: bool) -> None:
        dev = layer.w1.device
        comm = layer.comm
        C = ops.capacity(T, layer.top_k, layer.num_experts, layer.capacity_factor)
        if C < 1:
            raise InvalidPartitioningError(f"capacity {C} < 1 for T={T}")
        if not 1 <= n <= C:
            raise InvalidPartitioningError(f"pipeline granularity n={n} must be in [1, C={C}]")
        g = Geometry(T, layer.d_model, layer.d_hidden, layer.num_experts, comm.nranks, comm.rank, layer.top_k, C, n)
        self.layer, self.g, self.dtype, self.dev = layer, g, dtype, dev
        self.strategy = strategy
        self.reuse = reuse and n >= 2 and strategy.saves_memory
        self.timing = timing
        self.device_bytes = 0
        # reference memory categories (memmodel.py / engine.py:329-400): activations,
        # buffers (activation gradients), plus routing tensors and wgrad accumulators
        self.bytes_by_category: dict[str, int] = {}
        self.spec = ModelSpec(g.M, g.H, g.E, g.N, element_bytes=torch.empty((), dtype=dtype).element_size())
        self.batch = BatchSpec(g.E * C, n)
        E, k, M, H, N, e_loc = g.E, g.k, g.M, g.H, g.N, g.e_loc
        # routing
        self.logits = self._empty(T, E, dtype=torch.float32)
        self.idx = self._empty(T, k, dtype=torch.int32)
        self.weights = self._empty(T, k, dtype=torch.float32)
        self.slot = self._empty(T, k, dtype=torch.int32)
        self.kept = self._empty(E, dtype=torch.int32)
        self.route_ws = self._empty(max(int(_lib.load().mpm_route_workspace_bytes(T, E, k)), 16), dtype=torch.uint8)
        self.dprob = self._empty(T, k, dtype=torch.float32)
        self.dlogits = self._empty(T, E, dtype=torch.float32)
        self.routing = ops.Routing(self.logits, self.idx, self.weights, self.slot, self.kept, C, self.route_ws)
        # Padding skip (N = 1): slots fill in order, so chunk i of expert e holds a prefix of
        # rows[i][e] = clamp(kept[e] - s_i, 0, c_i) routed rows and zero padding after it.  The expert
        # GEMMs skip the all-padding row tiles and the weight gradients the padding K blocks.  At
        # N > 1 a capacity-layout chunk interleaves every source's padded block; the compacted expert
        # side below (fused dispatch) restores one routed prefix per expert.
        self.skip_padding = N == 1 and layer._skip_padding
        self.chunk_rows = self._empty(g.n_s, E, dtype=torch.int32) if self.skip_padding else None
        # dispatch-side full buffers (t_i, t_o, g_o, g_i pools); with the peer-memory
        # communicator they live in this arena's IPC window (with the gate-gradient
        # slices and the exchange flags), at the same offsets on every rank
        self.p2p = getattr(comm, "kind", None) == "p2p" and N > 1
        # Fused dispatch (peer memory, no reuse): senders gather their rows straight from the token
        # rows into the receivers' expert-side T_DI / g_do (window), so the dispatch-side T_I / g_o
        # (and their HBM round trip) do not exist.  With reuse the expert side is a ring of slots
        # that peers cannot target, so the dispatch pulls from T_I / g_o (and RC_i re-pulls T_I).
        self.fused = self.p2p and not self.reuse
        self.win = None
        self.flag_value = ctypes.c_uint32(1)  # every exchange flag is raised to 1 and reset to 0 (csrc/p2p.cu)
        self._p2p_keep: list = []
        self.t_i = self.g_o = None
        if self.p2p:
            esz = torch.empty((), dtype=dtype).element_size()
            self.wl = WindowLayout(N, E, C, M, esz, n, E * M, fused=self.fused)
            self.win = comm.window(self.wl.total)
            self.device_bytes += self.wl.total
            self.p2p_counters = self._empty(16 * n + 16, dtype=torch.int32)
            self.p2p_counters.zero_()
            names = (("t_di", "activations"), ("t_o", "activations"), ("g_do", "buffers"), ("g_i", "buffers")) \
                if self.fused else (("t_i", "activations"), ("t_o", "activations"), ("g_o", "buffers"),
                                    ("g_i", "buffers"))
            self.win_full: dict[str, torch.Tensor] = {}
            for name, cat in names:
                t_ = self.win.tensor(self.wl.off[name], (E * C, M), dtype)
                if name in ("t_di", "g_do"):
                    self.win_full[name] = t_.view(-1)  # expert-side [E_loc][N*C][M], peers push into it
                else:
                    setattr(self, name, t_)
                self.bytes_by_category[cat] = self.bytes_by_category.get(cat, 0) + E * C * M * esz
            self.bytes_by_category["routing"] = (self.bytes_by_category.get("routing", 0) + self.wl.total
                                                 - 4 * E * C * M * esz)
            self.win_name = {t_.data_ptr(): nm for nm, t_ in (("t_i", self.t_i), ("t_o", self.t_o),
                                                              ("g_o", self.g_o), ("g_i", self.g_i)) if t_ is not None}
            if self.fused:  # slot owners for the gathers, and the per-step source row pointers
                self.inv = self._empty(E * C, dtype=torch.int32)
                self.x_ptr, self.dy_ptr = _V(), _V()
        else:
            self.t_i = self._empty(E * C, M, cat="activations")
            self.t_o = self._empty(E * C, M, cat="activations")
            self.g_o = self._empty(E * C, M, cat="buffers")
            self.g_i = self._empty(E * C, M, cat="buffers")
        # Compacted expert side (fused dispatch, one slot part per expert group): every rank publishes
        # its kept[E] with its XS_FREE signal, each sender places its routed rows of expert e after the
        # lower sources' rows, so an expert's rows from all sources are one routed prefix (rows_compact)
        # and the capacity padding a single tail the GEMMs skip (valid rows / valid K) — the N > 1
        # counterpart of the N = 1 padding skip (capacity padding: ~2 % of the rows at cf 1.0, ~20 % at
        # cf 1.25); padding rows are no longer sent over NVLink either.
        # With memory reuse the expert side is a ring of slots that the receiver pulls into: the same
        # compaction per chunk slot range (mpm_compact_pull), the counts riding on TI_READY.
        self.compact = ((self.fused and g.n_s == 1) or (self.p2p and not self.fused)) and E % 4 == 0 \
            and layer._compact
        if self.compact:
            self.rows_compact = self._empty(n, g.e_loc, dtype=torch.int32)  # per chunk slot range
            self.kept_all = ("win", g.rank, self.wl.off["kept"])
        strat = self.strategy if self.reuse else NO_REUSE
        self.fw_dag = build_schedule(self.spec, self.batch, strat, self.reuse, FORWARD)
        self.bw_dag = build_schedule(self.spec, self.batch, strat, self.reuse, BACKWARD)
        caps = {**{k_: p.capacity for k_, p in self.fw_dag.pools.items()},
                **{k_: p.capacity for k_, p in self.bw_dag.pools.items()}}
        pools: dict[str, Pool] = {}
        self.full: dict[str, torch.Tensor] = {}  # all-chunk expert-side buffers (no ring)
        alias_of = {"t_di": self.t_i, "t_do": self.t_o, "g_do": self.g_o, "g_di": self.g_i}
        for name, width in (("t_di", M), ("t_m", H), ("t_do", M), ("g_do", M), ("g_m", H), ("g_di", M)):
            cat = "activations" if name.startswith("t_") else "buffers"
            if N == 1 and name in alias_of:
                self.full[name] = alias_of[name]
            elif self.fused and name in self.win_full:
                self.full[name] = self.win_full[name]
            elif not self.reuse:
                self.full[name] = self._empty(e_loc * N * C * width, cat=cat)
            if name in self.full:
                pools[name] = Pool(name, 1, alias=lambda i, b=self.full[name], w=width:
                                   _full_view(b, g, i, w, e_loc, N))
            else:
                pools[name] = Pool(name, caps[name], [self._empty(g.max_experts * g.max_rows * width, cat=cat)
                                                      for _ in range(caps[name])])
        self.pools = pools
        # 1-bit ReLU masks (bf16 path): fc1 / recompute write bit(T_M > 0) next to
        # T_M; fc2 dgrad reads 1/16 of T_M's bytes instead of T_M
        self.use_mask = dtype != torch.float32
        # mask rows padded to 16 bytes (4 words) so every chunk's view starts aligned for the
        # epilogue's vector stores (H/32 words per row otherwise, e.g. 5 at H=160)
        self.mask_w = -(-(H // 32) // 4) * 4
        self.masks: dict[int, torch.Tensor] = {}
        self.mask_full = None
        if self.use_mask:
            if "t_m" in self.full:
                self.mask_full = self._empty(e_loc * N * C * self.mask_w, dtype=torch.int32, cat="activations")
            else:
                for buf in pools["t_m"].buffers:
                    self.masks[buf.data_ptr()] = self._empty(g.max_experts * g.max_rows * self.mask_w,
                                                             dtype=torch.int32, cat="activations")
        # weight gradients: one GEMM over all chunks without reuse.  With reuse the rings are
        # overwritten, so each chunk computes its experts' weight gradient right after G2/G1: with
        # one slot part per expert group (n_s = 1, n <= E_loc) that is the expert's whole gradient
        # (stored once, one rounding); with n_s > 1 the parts of a group accumulate — in the
        # parameter dtype (one rounding per part, no scratch) or through fp32 accumulators
        # (wgrad_accumulation="fp32")
        self.deferred_wgrad = not self.reuse
        self.acc1 = self.acc2 = None
        if self.reuse and g.n_s > 1 and dtype != torch.float32 and layer.wgrad_accumulation == "fp32":
            self.acc1 = self._empty(*layer.w1.shape, dtype=torch.float32, cat="wgrad_accumulators")
            self.acc2 = self._empty(*layer.w2.shape, dtype=torch.float32, cat="wgrad_accumulators")
        # host slices for offload strategies (T_DI only when it is not an alias of T_I)
        self.host_di = self.host_m = self.host_mask = None
        if self.reuse and strat.restore_dispatched_input is RestoreMethod.OFFLOAD and "t_di" not in self.full:
            self.host_di = [layer._pinned(("di", T, n, i), g.chunk(i).ne * g.rows(i) * M, dtype) for i in range(n)]
        if self.reuse and strat.restore_middle is RestoreMethod.OFFLOAD:
            self.host_m = [layer._pinned(("m", T, n, i), g.chunk(i).ne * g.rows(i) * H, dtype) for i in range(n)]
            if self.use_mask:
                self.host_mask = [layer._pinned(("mask", T, n, i), g.chunk(i).ne * g.rows(i) * self.mask_w,
                                                torch.int32) for i in range(n)]
        # streams: mutable handles shared by every prebuilt call
        self.streams = {COMPUTE_STREAM: _V(), COLLECTIVE_STREAM: _V(layer._stream("collective").cuda_stream),
                        COPY_STREAM: _V(layer._stream("copy").cuda_stream)}
        # private gate workspace: arenas of different layers / ranks may run concurrently
        self.gate_ws = self._empty(int(_lib.load().mpm_gate_workspace_bytes(T, M, E)), dtype=torch.uint8)
        if self.p2p:  # "my T_I / g_o may be pulled" signals and the gate-gradient all-reduce
            cs = self.streams[COMPUTE_STREAM]
            if self.fused and self.compact:  # ... carrying this rank's kept counts (the compacted row offsets)
                self.xs_free = self._p2p_call(kept_signal_plan(self.wl, g.rank), {"kept": self.kept.data_ptr()}, cs)
            elif self.fused:  # "my expert-side buffers may be overwritten": raised at every forward start
                self.xs_free = self._p2p_call(signal_plan(self.wl, g.rank, FLAG_XS_FREE), {}, cs)
            else:
                self.ready_ti = (self._p2p_call(kept_signal_plan(self.wl, g.rank, FLAG_TI_READY),
                                                {"kept": self.kept.data_ptr()}, cs) if self.compact else
                                 self._p2p_call(signal_plan(self.wl, g.rank, FLAG_TI_READY), {}, cs))
                self.ready_go = self._p2p_call(signal_plan(self.wl, g.rank, FLAG_GO_READY), {}, cs)
            self.gate_stream = _V(layer._stream("gate").cuda_stream)
            if (E * M) % 4:
                raise InvalidPartitioningError("peer-memory gate all-reduce needs E*M % 4 == 0")
            self.dwg_reduce = self._p2p_call(reduce_plan(self.wl, g.rank, E * M * 4), {}, self.gate_stream)
            self.dwg_slice = self.win.tensor(self.wl.stage(g.rank), (E, M), torch.float32)
        # Compute lanes (B200): without reuse every chunk owns its expert-side rows, so consecutive
        # chunks' expert GEMMs are independent; odd chunks run on a second compute stream and one
        # chunk's GEMM fills the SMs the other's last partial wave leaves idle (the chunked GEMMs of
        # the N=8 shape: 486 -> 403 us at n=4, tools/chunk_gemm_probe.py).  With reuse the ring slots
        # are recycled across lanes behind the releasing ops' events (runtime.plan_dag), and with one
        # slot part per expert group (n_s = 1) the chunks' weight gradients touch disjoint experts, so
        # two lanes are safe too; only per-part accumulation (n_s > 1) keeps one lane (fixed add order).
        # Only for chunk GEMMs of a few dozen waves: the second lane fills a GEMM's last partial wave,
        # worth at most one wave in W. At BASELINE configs[3] (24576 pair tiles per chunk GEMM) the second lane
        # was 10 % slower (686 vs 617 ms per step, SM clock 780 vs 920 MHz under the power cap;
        # profiles/r2/r2cfg4_*).
        chunk_tiles = g.max_experts * -(-g.max_rows // 256) * -(-g.H // 256)
        self.lanes: dict[str, int] = {}
        if ((not self.reuse or g.n_s == 1) and n >= 2 and layer.compute_lanes >= 2
                and chunk_tiles <= LANE_MAX_TILES):
            self.streams["compute_b"] = _V(layer._stream("compute_b").cuda_stream)
            for dag_ in (self.fw_dag, self.bw_dag):
                for op_id, node in dag_.ops.items():
                    if node.stream == COMPUTE_STREAM and node.partition % 2 == 1:
                        self.lanes[op_id] = 1
        lane_streams = lambda dag_: {o: self.streams["compute_b"] for o in self.lanes if o in dag_.ops}  # noqa: E731
        # per-step pointers patched before issue
        self._keep: list[GemmArgs] = []
        self._fork_events: list = []
        self._wgrad_args: list[tuple[GemmArgs, str, int]] = []  # (args, weight, byte offset of its experts)
        self._dag = self.fw_dag
        self.fw_exec = PipelineExecutor(self.fw_dag, pools, self._calls, self.streams, timing,
                                        lanes=lane_streams(self.fw_dag))
        for p in pools.values():
            p.reset_ring()  # backward starts after the forward joined: every ring slot is free
        self._dag = self.bw_dag
        self.bw_exec = PipelineExecutor(self.bw_dag, pools, self._calls, self.streams, timing,
                                        lanes=lane_streams(self.bw_dag))
        self.wgrad_calls: list = []
        if self.deferred_wgrad:
            M_, H_ = M, H
            all_ = lambda name, w: self.full[name].reshape(e_loc, N * C, w)
            # K = every chunk's rows of the expert: kept (N = 1) or the compacted routed rows (N > 1)
            vk = self.kept if self.skip_padding else (self.rows_compact[0] if self.compact else None)
            self.wgrad_calls = [
                self._gemm(COMPUTE_STREAM, all_("g_do", M_), all_("t_m", H_), layer.w2, a_mn=True, b_mn=True,
                           valid_k=vk),
                self._gemm(COMPUTE_STREAM, all_("g_m", H_), all_("t_di", M_), layer.w1, a_mn=True, b_mn=True,
                           valid_k=vk),
            ]
            self._wgrad_args += [(self._keep[-2], "w2", 0), (self._keep[-1], "w1", 0)]
        self.origin = _lib.Event(True) if timing else None
        self.bw_origin = _lib.Event(True) if timing else None
        self.wgrad_events = (_lib.Event(True), _lib.Event(True)) if timing else None
        # phase boundaries of the last issue (timing arenas): fwd routing | DAG | combine,
        # bwd combine_bwd | DAG | (gather on the gate stream beside the deferred wgrad) | end
        self.marks = {k_: _lib.Event(True) for k_ in ("f0", "f1", "f2", "f3", "b0", "b1", "b2", "b3", "b4")} if timing else {}

    def _empty(self, *shape, dtype=None, cat: str = "routing") -> torch.Tensor:
        t = torch.empty(*shape, device=self.dev, dtype=dtype or self.dtype)
        if cat != "routing":
            t.zero_()  # padding rows of capacity blocks must read as zeros
        nbytes = t.numel() * t.element_size()
        self.device_bytes += nbytes
        self.bytes_by_category[cat] = self.bytes_by_category.get(cat, 0) + nbytes
        return t

    # ------------------------------------------------ op -> prebuilt C-ABI calls
    def _a2a(self, direction: int, pool: str, dispatch_buf: torch.Tensor, i: int, stream_name: str,
             redispatch: bool = False) -> list:
        """Chunk i's all-to-all between a dispatch-side buffer and an expert-side pool.

        Peer memory: a dispatch-type pull waits for the sources' ready flags (raised once per step
        after the permute / combine_bwd) and the last chunk's pull resets them; a re-dispatch
        (RC_i, S2/S4) reads rows the forward's pulls already waited for, so it does not wait."""
        g = self.g
        if g.N == 1:
            return []
        ch = g.chunk(i)
        c_i, s_i = ch.cs, ch.s0
        if pool in self.full:  # row of (expert e0, source 0, slot s0) in the all-chunk buffer
            expert_base, x_stride, x_row0 = self.full[pool], g.N * g.C, ch.e0 * g.N * g.C + g.N * s_i
        else:
            expert_base, x_stride, x_row0 = self.pools[pool].get(i), g.N * c_i, 0
        grp = dict(e0=ch.e0, ne=ch.ne)
        if self.fused and direction == _lib.A2A_DISPATCH:
            return self._push(pool, i, stream_name)
        if self.compact and direction == _lib.A2A_COMBINE:  # combine-type exchange, compacted expert side
            name = self.win_name[dispatch_buf.data_ptr()]
            slot = self.wl.r_slot(i) if name == "t_o" else self.wl.br_slot(i)
            plan = combine_push_plan(self.wl, g.rank, g.e_loc, g.C, c_i, s_i, name, slot, x_stride, x_row0, **grp)
            plan["kept_all"] = self.kept_all
            st = self.streams[stream_name]
            j = len(self._p2p_keep)
            if j >= self.p2p_counters.numel():
                raise RuntimeError("p2p counter block exhausted")
            lowered = lower_push(plan, self.win.bases, g.rank, self.p2p_counters[j:j + 1].data_ptr())
            self._p2p_keep.append(lowered)
            return [Call("mpm_combine_push", ctypes.byref(lowered), _V(expert_base.data_ptr()),
                         ops.dtype_code(self.dtype), g.M, self.flag_value, st),
                    self._p2p_call({"wait": [], "copy": [], "signal": [], "arrive": plan["arrive"],
                                    "reset": plan["reset"]}, {}, st)]
        if self.p2p and self.compact and direction == _lib.A2A_DISPATCH:  # reuse: pull into the ring
            return self._compact_pull(dispatch_buf, i, stream_name, expert_base, x_stride, x_row0, redispatch)
        if self.p2p:
            name = self.win_name[dispatch_buf.data_ptr()]
            loc = ("loc", "x", 0)
            if direction == _lib.A2A_DISPATCH:
                ready = None if redispatch else (FLAG_TI_READY if name == "t_i" else FLAG_GO_READY)
                plan = pull_plan(self.wl, g.rank, g.e_loc, g.C, c_i, s_i, name, ready, loc, x_stride, x_row0,
                                 reset=ready is not None and i == g.n - 1, **grp)
            else:
                slot = self.wl.r_slot(i) if name == "t_o" else self.wl.br_slot(i)
                plan = push_plan(self.wl, g.rank, g.e_loc, g.C, c_i, s_i, name, slot, loc, x_stride, x_row0, **grp)
            return [self._p2p_call(plan, {"x": expert_base.data_ptr()}, self.streams[stream_name])]
        plan = block_plan(direction, g.N, g.e_loc, c_i, g.M, g.C, s_i, x_stride, x_row0, **grp)
        src, dst = (dispatch_buf, expert_base) if direction == _lib.A2A_DISPATCH else (expert_base, dispatch_buf)
        comm = self.layer.comm
        if getattr(comm, "loopback", False):  # single-GPU multi-rank test harness
            stream = self.streams[stream_name]
            torch_stream = self.layer._stream("collective") if stream_name == COLLECTIVE_STREAM else None
            return [lambda: comm.a2a(direction, src, dst, plan, c_i * g.M,
                                     torch_stream or torch.cuda.current_stream())]
        peers, soff, roff = plan
        nb = len(peers)
        return [Call("mpm_a2a_chunk", self.layer.comm.handle, g.N, nb, (ctypes.c_int32 * nb)(*peers),
                     (ctypes.c_int64 * nb)(*soff), (ctypes.c_int64 * nb)(*roff), c_i * g.M,
                     ops.dtype_code(src.dtype), _V(src.data_ptr()), _V(dst.data_ptr()), self.streams[stream_name])]

    def _compact_pull(self, dispatch_buf: torch.Tensor, i: int, stream_name: str, expert_base: torch.Tensor,
                      x_stride: int, x_row0: int, redispatch: bool) -> list:
        """Dispatch-type pull of chunk i into the compacted expert-side rows (memory reuse): wait for
        every source's ready flag (TI_READY carries the kept counts), compute the chunk's routed rows
        per local expert (S_i), pull each source's routed rows to its prefix offset, reset the flags
        after the step's last pull."""
        g = self.g
        ch = g.chunk(i)
        st = self.streams[stream_name]
        name = self.win_name[dispatch_buf.data_ptr()]
        ready = None if redispatch else (FLAG_TI_READY if name == "t_i" else FLAG_GO_READY)
        waits = [] if ready is None else [("win", g.rank, self.wl.flag(ready, p)) for p in range(g.N) if p != g.rank]
        calls = []
        if waits:
            calls.append(self._p2p_call({"wait": waits, "copy": [], "signal": [], "arrive": [], "reset": []}, {}, st))
        if name == "t_i" and not redispatch:
            calls.append(Call("mpm_compact_rows", _V(self.win.addr(g.rank, self.wl.off["kept"])), g.N, g.E, g.e_loc,
                              g.rank, ch.s0, ch.cs, _V(self.rows_compact[i].data_ptr()), st))
        plan = compact_pull_plan(self.wl, g.rank, g.e_loc, g.C, ch.cs, ch.s0, name, x_stride, x_row0,
                                 e0=ch.e0, ne=ch.ne)
        plan["kept_all"] = self.kept_all
        lowered = lower_push(plan, self.win.bases, g.rank, 0)
        self._p2p_keep.append(lowered)
        calls.append(Call("mpm_compact_pull", ctypes.byref(lowered), _V(expert_base.data_ptr()),
                          ops.dtype_code(self.dtype), g.M, st))
        if waits and i == g.n - 1:  # the step's last wait on these flags
            calls.append(self._p2p_call({"wait": [], "copy": [], "signal": [], "arrive": [], "reset": waits}, {}, st))
        return calls

    def _push(self, pool: str, i: int, stream_name: str) -> list:
        """Fused dispatch of chunk i (S_i: token rows x; BS_i: routed gradients w * dy): gather this
        rank's rows into every destination's expert-side buffer (mpm_dispatch_push), then wait for
        every peer's rows of the chunk here.  S_0 first waits until every destination has released
        its expert-side buffers from the previous step (XS_FREE, raised at its forward start)."""
        g = self.g
        ch = g.chunk(i)
        st = self.streams[stream_name]
        grad = pool == "g_do"
        slot = self.wl.bs_slot(i) if grad else self.wl.s_slot(i)
        plan = push_dispatch_plan(self.wl, g.rank, g.e_loc, g.C, ch.cs, ch.s0, pool, slot, e0=ch.e0, ne=ch.ne)
        if self.compact:
            plan["kept_all"] = self.kept_all
        calls = []
        if i == 0 and not grad:
            free = [("win", g.rank, self.wl.flag(FLAG_XS_FREE, p)) for p in range(g.N) if p != g.rank]
            calls.append(self._p2p_call({"wait": free, "copy": [], "signal": [], "arrive": [], "reset": free},
                                        {}, st))
            if self.compact:  # every source's counts are here now: the local experts' routed rows
                calls.append(Call("mpm_compact_rows", _V(self.win.addr(g.rank, self.wl.off["kept"])), g.N, g.E,
                                  g.e_loc, g.rank, 0, g.C, _V(self.rows_compact[0].data_ptr()), st))
        j = len(self._p2p_keep)
        if j >= self.p2p_counters.numel():
            raise RuntimeError("p2p counter block exhausted")
        lowered = lower_push(plan, self.win.bases, g.rank, self.p2p_counters[j:j + 1].data_ptr())
        self._p2p_keep.append(lowered)
        src = self.dy_ptr if grad else self.x_ptr
        scale = _V(self.weights.data_ptr()) if grad else _V(None)
        calls.append(Call("mpm_dispatch_push", ctypes.byref(lowered), src, ops.dtype_code(self.dtype), g.M, g.k,
                          _V(self.inv.data_ptr()), scale, self.flag_value, st))
        calls.append(self._p2p_call({"wait": [], "copy": [], "signal": [], "arrive": plan["arrive"],
                                     "reset": plan["reset"]}, {}, st))
        return calls

    def _p2p_call(self, plan: dict, locals_: dict, stream) -> Call:
        # every plan owns one zeroed uint32 of the arena's counter block (SM copy completion count)
        j = len(self._p2p_keep)
        if j >= self.p2p_counters.numel():
            raise RuntimeError("p2p counter block exhausted")
        lowered = lower_plan(plan, self.win.bases, locals_, self.p2p_counters[j:j + 1].data_ptr())
        self._p2p_keep.append(lowered)  # the struct must outlive its byref in the prebuilt call
        return Call("mpm_p2p_run", ctypes.byref(lowered), self.flag_value, stream)

    def _gemm(self, stream_name: str, *a, **kw) -> Call:
        args = _gemm_args(*a, **kw)
        self._keep.append(args)  # the struct must outlive its byref in the prebuilt call
        return Call("mpm_grouped_gemm", ctypes.byref(args), self.streams[stream_name])

    def _copy(self, dst: torch.Tensor, src: torch.Tensor, direction: int, stream_name: str) -> Call:
        return Call("mpm_copy_async", _V(dst.data_ptr()), _V(src.data_ptr()), src.numel() * src.element_size(),
                    direction, self.streams[stream_name])

    def view(self, pool: str, i: int, width: int) -> torch.Tensor:
        p = self.pools[pool]
        return p.get(i) if p.alias is not None else _ring_view(p.get(i), self.g, i, width)

    def mask_view(self, i: int) -> torch.Tensor:
        g = self.g
        if self.mask_full is not None:
            return _full_view(self.mask_full, g, i, self.mask_w, g.e_loc, g.N)
        return _ring_view(self.masks[self.pools["t_m"].get(i).data_ptr()], g, i, self.mask_w)

    def _calls(self, op_id: str) -> list:
        g, lay = self.g, self.layer
        node = self._dag.ops[op_id]
        i, st = node.partition, ("compute_b" if op_id in self.lanes else node.stream)
        M, H = g.M, g.H
        view = lambda pool, w: self.view(pool, i, w)
        relu_epi = _lib.EPI_RELU_MASK if self.use_mask else _lib.EPI_RELU
        relu_aux = (lambda: self.mask_view(i)) if self.use_mask else (lambda: None)
        ch = g.chunk(i)
        ex = slice(ch.e0, ch.e0 + ch.ne)  # the chunk's local experts
        w1, w2 = lay.w1[ex], lay.w2[ex]
        # routed rows of each of the chunk's experts in its slot part (padding skip: N = 1, or the
        # compacted expert side at N > 1)
        vr = self.chunk_rows[ch.part, ex] if self.skip_padding else (
            (self.rows_compact[0 if self.fused else i, ex]) if self.compact else None)
        if op_id.startswith("RC"):
            return self._a2a(_lib.A2A_DISPATCH, "t_di", self.t_i, i, st, redispatch=True)
        if op_id[0] == "S":
            return self._a2a(_lib.A2A_DISPATCH, "t_di", self.t_i, i, st)
        if op_id[0] == "C":
            t_di, t_m = view("t_di", M), view("t_m", H)
            return [self._gemm(st, t_di, w1, t_m, epilogue=relu_epi, aux=relu_aux(), valid_rows=vr),
                    self._gemm(st, t_m, w2, view("t_do", M), valid_rows=vr)]
        if op_id[0] == "R" and not op_id.startswith("RE"):
            return self._a2a(_lib.A2A_COMBINE, "t_do", self.t_o, i, st)
        if op_id.startswith("Ddi"):
            return [] if self.host_di is None else [self._copy(self.host_di[i], view("t_di", M), _lib.COPY_D2H, st)]
        if op_id.startswith("Dm"):
            calls = [self._copy(self.host_m[i], view("t_m", H), _lib.COPY_D2H, st)]
            if self.use_mask:
                calls.append(self._copy(self.host_mask[i], self.mask_view(i), _lib.COPY_D2H, st))
            return calls
        if op_id.startswith("BS"):
            return self._a2a(_lib.A2A_DISPATCH, "g_do", self.g_o, i, st)
        if op_id.startswith("Hdi"):
            return [] if self.host_di is None else [self._copy(view("t_di", M), self.host_di[i], _lib.COPY_H2D, st)]
        if op_id.startswith("Hm"):
            calls = [self._copy(view("t_m", H), self.host_m[i], _lib.COPY_H2D, st)]
            if self.use_mask:
                calls.append(self._copy(self.mask_view(i), self.host_mask[i], _lib.COPY_H2D, st))
            return calls
        if op_id.startswith("RE"):
            return [self._gemm(st, view("t_di", M), w1, view("t_m", H), epilogue=relu_epi, aux=relu_aux(),
                               valid_rows=vr)]
        if op_id.startswith("G2_"):
            g_do, t_m, g_m = view("g_do", M), view("t_m", H), view("g_m", H)
            if self.use_mask:
                calls = [self._gemm(st, g_do, w2, g_m, b_mn=True, epilogue=_lib.EPI_DMASK, aux=self.mask_view(i),
                                    valid_rows=vr)]
            else:
                calls = [self._gemm(st, g_do, w2, g_m, b_mn=True, epilogue=_lib.EPI_DRELU, aux=t_m, valid_rows=vr)]
            if not self.deferred_wgrad:
                return self._forked(st, calls, [self._wgrad(self._side(st), g_do, t_m, lay.w2, self.acc2, i, "w2", vr)])
            return calls
        if op_id.startswith("G1_"):
            g_m, t_di, g_di = view("g_m", H), view("t_di", M), view("g_di", M)
            calls = [self._gemm(st, g_m, w1, g_di, b_mn=True, valid_rows=vr)]
            if not self.deferred_wgrad:
                return self._forked(st, calls, [self._wgrad(self._side(st), g_m, t_di, lay.w1, self.acc1, i, "w1", vr)])
            return calls
        if op_id.startswith("BR"):
            return self._a2a(_lib.A2A_COMBINE, "g_di", self.g_i, i, st)
        raise RuntimeError(f"no realisation for op {op_id}")  # pragma: no cover

    def _side(self, st: str) -> str:
        """The weight-gradient side stream of compute lane `st` (created on first use)."""
        name = "wgrad_b" if st == "compute_b" else "wgrad_a"
        if name not in self.streams:
            self.streams[name] = _V(self.layer._stream(name).cuda_stream)
        return name

    def _forked(self, st: str, main: list, side: list) -> list:
        """One DAG op whose calls fork: `side` (a chunk's weight-gradient GEMM) runs on the lane's side
        stream beside `main` (the dgrad GEMM that reads the same chunk rows); the op ends when both
        have (fork / join events), so the DAG's dependencies and slot releases are unchanged.  The
        two GEMMs fill each other's partial last waves (chunk GEMMs with few tiles per SM)."""
        fork, join = _lib.Event(False), _lib.Event(False)
        self._fork_events += [fork, join]
        a, b = self.streams[st], self.streams[self._side(st)]
        return [Call("mpm_event_record", fork.handle, a), Call("mpm_stream_wait", b, fork.handle), *side, *main,
                Call("mpm_event_record", join.handle, b), Call("mpm_stream_wait", a, join.handle)]

    def _wgrad(self, st, a, b, w, acc, i, which, valid_k=None) -> Call:
        """Chunk i's weight-gradient GEMM (reuse mode) for its experts; the grad pointer is patched
        per step.  The first slot part of an expert group stores, later parts accumulate (in the
        parameter dtype, or through the fp32 accumulators); with one part per group (n <= E_loc)
        every expert's gradient is one GEMM, stored once."""
        ch, n_s = self.g.chunk(i), self.g.n_s
        ex = slice(ch.e0, ch.e0 + ch.ne)
        first, last = ch.part == 0, ch.part == n_s - 1
        if acc is None:  # in place in the parameter dtype (TMA reduce-add after the first part)
            c, epi, aux = w[ex], (_lib.EPI_NONE if first else _lib.EPI_ACCUM), None
        elif first:
            c, epi, aux = acc[ex], _lib.EPI_STORE_F32, None
        elif not last:
            c, epi, aux = acc[ex], _lib.EPI_ACCUM_F32, None
        else:
            c, epi, aux = w[ex], _lib.EPI_ADD_AUX_F32, acc[ex]
        call = self._gemm(st, a, b, c, a_mn=True, b_mn=True, epilogue=epi, aux=aux, valid_k=valid_k)
        if c.data_ptr() != (acc[ex].data_ptr() if acc is not None else -1):
            # built against the parameter; the real target is the per-step grad tensor (same offset)
            self._wgrad_args.append((self._keep[-1], which, c.data_ptr() - w.data_ptr()))
        return call

    # ----------------------------------------------------------- issue
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """Issue the forward on the current stream; returns y (a fresh tensor)."""
        g, lay = self.g, self.layer
        compute = torch.cuda.current_stream()
        self.streams[COMPUTE_STREAM].value = compute.cuda_stream
        cs = self.streams[COMPUTE_STREAM]
        mark = (lambda k_: self.marks[k_].record(cs)) if self.marks else (lambda k_: None)
        if self.origin is not None:
            self.origin.record(cs)
        mark("f0")
        ops.gate_route(x, lay.gate_weight, g.k, lay.renorm, out=(self.logits, self.idx, self.weights, self.route_ws),
                       gate_ws=self.gate_ws)
        ops.assign_slots(self.idx, g.E, g.C, self.route_ws, out=(self.slot, self.kept))
        if self.skip_padding:
            _lib.call("mpm_chunk_rows", _V(self.kept.data_ptr()), g.E, g.C, g.n_s, _V(self.chunk_rows.data_ptr()),
                      cs)
        if self.fused:  # no T_I: the S_i pushes gather x rows through the slot-owner map
            self.x_ptr.value = x.data_ptr()
            _lib.call("mpm_slot_owners", _V(self.idx.data_ptr()), _V(self.slot.data_ptr()), _V(self.kept.data_ptr()),
                      g.T, g.E, g.k, g.C, _V(self.inv.data_ptr()), cs)
            self.xs_free()
        else:
            ops.permute(x, self.routing, g.n, self.t_i)
            if self.p2p:
                self.ready_ti()
        mark("f1")
        self.fw_exec.run(cs)
        self.fw_exec.join(cs)
        if self.p2p:
            self.watch(cs.value, "MoELayer forward exchanges")
        mark("f2")
        y = ops.combine(self.t_o, self.routing, g.n, g.T)
        mark("f3")
        return y

    def backward(self, x: torch.Tensor, dy: torch.Tensor):
        """Issue the backward; returns fresh (dx, dwg, dw1, dw2)."""
        g, lay = self.g, self.layer
        compute = torch.cuda.current_stream()
        cs = self.streams[COMPUTE_STREAM]
        cs.value = compute.cuda_stream
        mark = (lambda k_: self.marks[k_].record(cs)) if self.marks else (lambda k_: None)
        if self.bw_origin is not None:
            self.bw_origin.record(cs)
        mark("b0")
        # Combine + gate backward.  One pass per token (combine_bwd_gate) yields the g_o rows, dprob,
        # dlogits and the split operands of the gate GEMMs; then dWg (and, for a dense gate gradient,
        # the gate term of dx).  Single rank: all of it on the compute stream ahead of the expert
        # backward — the gate GEMMs are tcgen05 kernels that cannot share an SM with the persistent
        # expert GEMMs, and HBM kernels beside them only trade GEMM time for their own (measured:
        # tools/overlap_ab.py, tools/kernel_timeline.py).  Peer memory (N > 1): the dispatch side
        # (g_o, or the fused BS_i pushes) stays on the compute stream and the gate part runs on the
        # gate stream under the expert backward, followed by the gate-gradient all-reduce (push
        # slices, fixed-rank-order sum).
        dx = torch.empty_like(x)  # the gate term lands here first (dense case); the gather writes the rest
        gs = lay._stream("gate")
        if self.p2p:
            gs.wait_stream(compute)
            if self.fused:  # no g_o: the BS_i pushes gather w * dy rows through the slot-owner map
                self.dy_ptr.value = dy.data_ptr()
            else:
                ops.combine_bwd(dy, self.t_o, self.routing, g.n, self.g_o, dprob=False)
                self.ready_go()
            mark("b1")
            ops.combine_bwd_gate(dy, self.t_o, self.routing, g.n, None, self.dlogits, self.gate_ws, lay.renorm,
                                 dprob=self.dprob, stream=gs)
            ops.gate_backward_gemms(x, lay.gate_weight, self.dlogits, g.k, lay.renorm, self.dwg_slice, dx,
                                    self.gate_ws, stream=gs)
            self.dwg_reduce()
            dwg = torch.empty(g.E, g.M, device=self.dev, dtype=torch.float32)
            _lib.call("mpm_sum_slices", _V(self.win.addr(g.rank, self.wl.stage(0))), g.N,
                      self.wl.stage_slice // 4, g.E * g.M, _V(dwg.data_ptr()), self.gate_stream)
        else:
            ops.combine_bwd_gate(dy, self.t_o, self.routing, g.n, self.g_o, self.dlogits, self.gate_ws, lay.renorm,
                                 dprob=self.dprob)
            dwg = torch.empty(g.E, g.M, device=self.dev, dtype=torch.float32)
            ops.gate_backward_gemms(x, lay.gate_weight, self.dlogits, g.k, lay.renorm, dwg, dx, self.gate_ws)
            mark("b1")
        dw1 = torch.empty_like(lay.w1)
        dw2 = torch.empty_like(lay.w2)
        for args, which, off in self._wgrad_args:
            args.c = (dw1 if which == "w1" else dw2).data_ptr() + off
        self.bw_exec.run(cs)
        # The gather needs only g_i (complete once every stream's last DAG op is done) and the gate
        # term already in dx (gate stream): it runs on the gate stream beside the deferred
        # weight-gradient GEMMs (no shared memory, so its CTAs fit next to the GEMM's).
        gsv = _V(gs.cuda_stream)
        gmark = (lambda k_: self.marks[k_].record(gsv)) if self.marks else (lambda k_: None)

        def gather():
            self.bw_exec.join(gsv)
            gmark("b2")
            ops.gate_gather(self.routing, self.g_i, lay.gate_weight, g.n, self.dlogits, lay.renorm, dx, self.gate_ws,
                            stream=gs)
            gmark("b3")

        if lay._gather_side:
            gather()
        if self.wgrad_calls:  # after the last G1 on the compute stream, overlapping the last BR
            if self.lanes:  # and after the last G1 of the other compute lane
                self.bw_exec.join(cs, only=[self.streams["compute_b"]])
            if self.wgrad_events:
                self.wgrad_events[0].record(cs)
            for c in self.wgrad_calls:
                c()
            if self.wgrad_events:
                self.wgrad_events[1].record(cs)
        self.bw_exec.join(cs)
        if not lay._gather_side:
            gather()
        compute.wait_stream(gs)
        if self.p2p:
            self.watch(cs.value, "MoELayer backward exchanges")
        mark("b4")
        if g.N > 1 and not self.p2p:
            lay.comm.all_reduce(dwg)  # the replicated gate is data parallel
        return dx, dwg, dw1, dw2

    def watch(self, stream: int, tag: str) -> None:
        """Arm the exchange watchdog behind the work issued so far (peer-memory arenas): a dead or
        stalled peer aborts this rank after MPM_WATCHDOG_TIMEOUT_S (default 300 s, 0 = off) instead
        of leaving its flag waits blocked forever."""
        timeout = float(os.environ.get("MPM_WATCHDOG_TIMEOUT_S", "300"))
        if timeout > 0:
            _lib.call("mpm_watchdog_watch", _V(stream), timeout,
                      f"{tag} (rank {self.g.rank} of {self.g.N}, T={self.g.T}, n={self.g.n})".encode())

    def phase_ms(self) -> dict:
        """Device time per phase of the last issue (timing arenas; synchronises)."""
        if not self.marks:
            return {}
        m = self.marks
        d = lambda a, b: round(m[a].elapsed_ms(m[b]), 4)
        return {"fwd_routing_permute": d("f0", "f1"), "fwd_dag": d("f1", "f2"), "fwd_combine": d("f2", "f3"),
                "bwd_combine_bwd": d("b0", "b1"), "bwd_dag": d("b1", "b2"),
                "bwd_gather_beside_wgrad": d("b2", "b3"), "bwd_dag_wgrad_gate": d("b1", "b4"),
                "fwd_total": d("f0", "f3"), "bwd_total": d("b0", "b4")}

    def wgrad_seconds(self) -> float:
        """Device time of the deferred weight-gradient GEMMs of the last backward (timing arenas)."""
        if not (self.wgrad_events and self.wgrad_calls):
            return 0.0
        return self.wgrad_events[0].elapsed_ms(self.wgrad_events[1]) * 1e-3

    def traces(self):
        """Measured (forward, backward) ScheduleTraces of the last issue (synchronises)."""
        from .trace import trace_from_times
        return (trace_from_times(self.fw_dag, self.fw_exec.times(), self.lanes),
                trace_from_times(self.bw_dag, self.bw_exec.times(), self.lanes))


class _MoEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, gate_weight, w1, w2, lease: "_Lease"):
        y = lease.arena.forward(x)
        ctx.lease = lease
        ctx.save_for_backward(x)
        return y

    @staticmethod
    def backward(ctx, dy):
        (x,) = ctx.saved_tensors
        lease = ctx.lease
        dx, dwg, dw1, dw2 = lease.arena.backward(x, dy.contiguous())
        lease.release()
        ctx.lease = None
        return dx, dwg, dw1, dw2, None


class _Lease:
    """An arena checked out for one in-flight step; returned after its backward
    (or when the autograd graph holding it is dropped without one)."""

    def __init__(self, layer: "MoELayer", key, arena: _Arena) -> None:
        self.arena = arena
        self._fin = weakref.finalize(self, layer._return_arena, key, arena)

    def release(self) -> None:
        self._fin()


class MoELayer(nn.Module):
    """Pipelined expert-parallel MoE FFN layer (tcgen05 experts; chunk exchanges over NVLink peer
    memory, or NCCL send/recv).

    Args:
      d_model, d_hidden, num_experts, top_k: layer shape.
      capacity_factor: C = ceil(cf * T * k / E) slots per (source rank, expert).
      pipeline: int n, "adaptive" / True (Algorithm 1), or False (n = 1).
      memory_reuse: False/"none", True/"auto" (runtime strategy selection),
        or one of "s1".."s4" (Table II).
      renorm: renormalise the top-k weights when k > 1.
      group: torch.distributed group of the expert-parallel ranks (None:
        the default group when initialised, else a single rank).
      dtype: expert weight / activation dtype (bf16 -> tcgen05; fp32 ->
        exact-fp32 kernels).
      max_cached_arenas: idle step arenas kept for reuse (one per token count /
        n / strategy); older ones are dropped when a new one is built.
      a2a_backend: "p2p" (exchanges over NVLink peer memory with one light
        copy kernel each, co-resident with the GEMMs; csrc/p2p.cu) or "nccl"
        (grouped ncclSend/Recv, the baseline).
      compute_lanes: 2 runs the expert GEMMs of odd chunks on a second compute
        stream when chunks are independent (no reuse, n >= 2); 1 keeps the
        reference's single compute stream (env MPM_COMPUTE_LANES overrides).
      wgrad_accumulation: with memory reuse each chunk's weight gradient is
        accumulated into dW: "param" (in the parameter dtype, one rounding
        per chunk, no scratch) or "fp32" (fp32 accumulators, one rounding;
        2x the expert weights' element count in fp32 scratch).
    All EP ranks must pass the same token count per step (symmetric
    capacity blocks, as the reference's per-device model assumes).
    """

    def __init__(self, d_model: int, d_hidden: int, num_experts: int, top_k: int = 1,
                 capacity_factor: float = 1.0, pipeline=True, memory_reuse=False, renorm: bool = True,
                 group=None, dtype: torch.dtype = torch.bfloat16, device=None,
                 candidates=(1, 2, 4, 8, 16), trials_per_candidate: int = 1, min_micro_batch: int = 1,
                 hw_profile=None, seed: int = 0, comm=None, wgrad_accumulation: str = "param",
                 a2a_backend: str = "p2p", max_cached_arenas: int = 4, compute_lanes: int = 2) -> None:
        super().__init__()
        if wgrad_accumulation not in ("param", "fp32"):
            raise ValueError(f"wgrad_accumulation must be 'param' or 'fp32', got {wgrad_accumulation!r}")
        if dtype == torch.bfloat16 and (d_model % 32 or d_hidden % 32):
            # the tcgen05 expert GEMMs emit 32-column epilogue slices (N = d_hidden for fc1, d_model for fc2)
            raise ValueError(f"bf16 experts need d_model and d_hidden multiples of 32 (got {d_model}, {d_hidden})")
        if dtype not in (torch.bfloat16, torch.float32):
            raise ValueError(f"expert dtype must be bfloat16 or float32, got {dtype}")
        self.wgrad_accumulation = wgrad_accumulation
        self.compute_lanes = int(os.environ.get("MPM_COMPUTE_LANES", compute_lanes))
        self.d_model, self.d_hidden, self.num_experts = d_model, d_hidden, num_experts
        self.top_k, self.capacity_factor, self.renorm = top_k, capacity_factor, renorm
        self.group = group
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.comm = comm if comm is not None else make_comm(a2a_backend, group, device)
        N = self.comm.nranks
        if num_experts % N:
            raise ValueError(f"num_experts ({num_experts}) must be divisible by the EP size ({N})")
        e_loc = num_experts // N
        self.gate_weight = nn.Parameter(torch.empty(num_experts, d_model, device=device, dtype=torch.float32))
        self.w1 = nn.Parameter(torch.empty(e_loc, d_hidden, d_model, device=device, dtype=dtype))
        self.w2 = nn.Parameter(torch.empty(e_loc, d_model, d_hidden, device=device, dtype=dtype))
        self.reset_parameters(seed)

        if pipeline is True or pipeline == "adaptive":
            self.pipeline = "adaptive"
        elif pipeline is False or pipeline is None:
            self.pipeline = 1
        else:
            self.pipeline = int(pipeline)
        if memory_reuse is True:
            memory_reuse = "auto"
        if memory_reuse in (False, None):
            memory_reuse = "none"
        memory_reuse = str(memory_reuse).lower()
        if memory_reuse not in ("none", "auto", "s1", "s2", "s3", "s4"):
            raise ValueError(f"memory_reuse must be none|auto|s1..s4, got {memory_reuse!r}")
        self.memory_reuse = memory_reuse
        self.candidates = tuple(candidates)
        self.trials_per_candidate = trials_per_candidate
        self.min_micro_batch = min_micro_batch
        self.hw_profile = hw_profile
        self._controller = None
        self._loaded_index = None
        self._streams: dict[str, torch.cuda.Stream] = {}
        self._pinned_cache: dict = {}
        self._arenas: dict = {}
        self.max_cached_arenas = max_cached_arenas
        self.record_times = False
        self.last_arena: _Arena | None = None
        self._skip_padding = True  # N = 1: skip capacity-padding row tiles / K blocks (A/B tools flip it)
        # N > 1 (fused dispatch): compacted expert side; MPM_COMPACT=0 keeps the capacity layout (A/B)
        self._compact = os.environ.get("MPM_COMPACT", "1") != "0"
        # the gather beside the deferred weight gradients on the gate stream, or after them
        # (A/B tools flip it: tools/overlap_ab.py)
        self._gather_side = True

    # ------------------------------------------------------------ plumbing
    def reset_parameters(self, seed: int = 0) -> None:
        """Synthetic init: W_g ~ N(0, 1/M) (seed 7), W1/W2 ~ N(0, 0.02^2) (seed 11+rank)."""
        with torch.no_grad():
            gen = torch.Generator(device="cpu").manual_seed(7 + seed)
            self.gate_weight.copy_(torch.randn(self.gate_weight.shape, generator=gen) / math.sqrt(self.d_model))
            gen = torch.Generator(device="cpu").manual_seed(11 + self.comm.rank + seed)
            self.w1.copy_(torch.randn(self.w1.shape, generator=gen) * 0.02)
            self.w2.copy_(torch.randn(self.w2.shape, generator=gen) * 0.02)

    def _stream(self, name: str) -> torch.cuda.Stream:
        if name not in self._streams:
            self._streams[name] = torch.cuda.Stream(device=self.w1.device)
        return self._streams[name]

    def _pinned(self, key, numel: int, dtype) -> torch.Tensor:
        t = self._pinned_cache.get(key)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(numel, dtype=dtype, pin_memory=True)
            self._pinned_cache[key] = t
        return t[:numel]

    def _checkout(self, T: int, n: int, strategy: ReuseStrategy, reuse: bool) -> tuple:
        key = (T, n, strategy.name, bool(reuse), self.w1.dtype, self.record_times, self.wgrad_accumulation)
        free = self._arenas.setdefault(key, [])
        if free:
            arena = free.pop()
        else:
            self._evict_idle()
            arena = _Arena(self, T, n, strategy, reuse, self.w1.dtype, self.record_times)
        self._arenas[key] = self._arenas.pop(key)  # most recently used key last
        return key, arena

    def _evict_idle(self) -> None:
        """Bound the idle-arena cache (dynamic batch sizes create one arena per token count):
        before building a new arena, drop the least recently used idle ones beyond
        `max_cached_arenas`.

        With the peer-memory communicator the eviction is collective: every EP rank passes the
        same token count in the same order (symmetric capacity blocks), so the LRU order of the
        keys — and therefore the victims — is identical on every rank, and their windows are
        unmapped and freed together here (Window.close is collective)."""
        idle = [(k_, a) for k_, lst in self._arenas.items() for a in lst]
        victims = idle[:max(0, len(idle) - self.max_cached_arenas + 1)]
        for k_, a in victims:
            self._arenas[k_].remove(a)
        windows = [a.win for _, a in victims if a.win is not None]
        if windows:
            self.comm.free(windows)

    def _return_arena(self, key, arena: _Arena) -> None:
        self._arenas.setdefault(key, []).append(arena)

    def release_arenas(self) -> None:
        """Drop every idle step arena (device memory back to the allocator).

        With the peer-memory communicator this is collective: the idle arenas'
        windows are unmapped and freed on every rank in the same order."""
        windows = [a.win for free in self._arenas.values() for a in free if a.win is not None]
        self._arenas.clear()
        if windows:
            self.comm.free(windows)

    # ------------------------------------------------------------ planning
    def capacity(self, tokens: int) -> int:
        return ops.capacity(tokens, self.top_k, self.num_experts, self.capacity_factor)

    def model_spec(self, element_bytes: int | None = None) -> ModelSpec:
        return ModelSpec(self.d_model, self.d_hidden, self.num_experts, self.comm.nranks,
                         element_bytes or self.w1.element_size())

    def hardware_profile(self, tokens: int | None = None):
        """The measured HardwareProfile (calibrated once, at `tokens` tokens per rank when given)."""
        if self.hw_profile is None:
            from .calibrate import measure_profile
            self.hw_profile = measure_profile(self, tokens=tokens)
        return self.hw_profile

    def plan(self, tokens: int) -> tuple[int, ReuseStrategy, bool]:
        """(n, strategy, reuse_enabled) for a batch of `tokens` tokens on this rank."""
        C = self.capacity(tokens)
        if self.pipeline == "adaptive":
            n = self._adaptive_n(tokens)
        else:
            n = max(1, min(self.pipeline, C))
        strategy = NO_REUSE
        if self.memory_reuse == "auto" and n >= 2:
            from .cost import select_strategy
            strategy = select_strategy(self.model_spec(), self.hardware_profile(tokens),
                                       math.ceil(self.num_experts * C / n)).strategy
        elif self.memory_reuse not in ("none", "auto"):
            strategy = ReuseStrategy.by_name(self.memory_reuse)
        return n, strategy, strategy.saves_memory and n >= 2

    def _adaptive_n(self, tokens: int) -> int:
        if self._controller is None:
            from .calibrate import GpuMeasurementAdapter
            from .granularity import AdaptiveController, TrialBudget
            budget = TrialBudget(self.candidates, self.trials_per_candidate, GpuMeasurementAdapter(self),
                                 self.min_micro_batch)
            strategy = NO_REUSE if self.memory_reuse in ("none", "auto") else ReuseStrategy.by_name(self.memory_reuse)
            self._controller = AdaptiveController(self.model_spec(), None, strategy, budget)
            if self._loaded_index is not None:  # resume Algorithm 1 from a checkpoint
                self._controller.index = self._loaded_index
                self._loaded_index = None
        searches = self._controller.stats.searches
        n = self._controller.adaptive_granularity(tokens * self.top_k)
        if self._controller.stats.searches != searches:
            self.release_arenas()  # drop the trial arenas of the candidates not chosen
            close = getattr(self._controller.budget.adapter, "close", None)
            if close is not None:
                close()  # and the search's anchor step graph
        return max(1, min(n, self.capacity(tokens)))

    # ------------------------------------------------------- checkpoint / resume
    def get_extra_state(self) -> dict:
        """Runtime-learned state saved with state_dict(): Algorithm 1's range index and cache
        (the reference keeps them in memory only, autotune.py:132-139) and the measured
        HardwareProfile, so a restarted job neither re-searches nor re-calibrates."""
        from .cli import profile_to_json
        state = {"version": 1}
        index = self._controller.index if self._controller is not None else self._loaded_index
        if index is not None:
            state["granularity_index"] = index.to_json()
        if self.hw_profile is not None:
            state["hw_profile"] = profile_to_json(self.hw_profile)
        return state

    def set_extra_state(self, state) -> None:
        from .cli import profile_from_json
        from .granularity import GranularityIndex
        if not state:
            return
        if "granularity_index" in state:
            index = GranularityIndex.from_json(state["granularity_index"])
            if self._controller is not None:
                self._controller.index = index
            else:
                self._loaded_index = index
        if "hw_profile" in state:
            self.hw_profile = profile_from_json(state["hw_profile"])

    # ------------------------------------------------------------ forward
    def run_step(self, x: torch.Tensor, dy: torch.Tensor, n: int, strategy: ReuseStrategy):
        """Forward + backward without autograd: (y, (dx, dwg, dw1, dw2)).

        Used by the measurement adapter, benchmarks and multi-rank harnesses
        (autograd runs every backward of a device on one engine thread, so
        lock-stepped ranks in one process cannot use it)."""
        reuse = strategy.saves_memory and n >= 2
        key, arena = self._checkout(x.shape[0], n, strategy, reuse)
        self.last_arena = arena
        try:
            y = arena.forward(x)
            grads = arena.backward(x, dy)
        finally:
            self._return_arena(key, arena)
        return y, grads

    def step_graph(self, tokens: int, n: int, strategy: ReuseStrategy) -> "StepGraph":
        """A CUDA graph of one forward + backward at a fixed token count (see StepGraph)."""
        return StepGraph(self, tokens, n, strategy)

    def forward(self, x: torch.Tensor, n: int | None = None, strategy: str | None = None) -> torch.Tensor:
        if not x.is_cuda:
            raise ValueError("MoELayer runs on CUDA only (no CPU path)")
        shape = x.shape
        x2 = x.reshape(-1, self.d_model)
        if x2.dtype != self.w1.dtype:
            raise TypeError(f"x dtype {x2.dtype} != expert dtype {self.w1.dtype}")
        x2 = x2.contiguous()
        if n is None:
            n, strat, reuse = self.plan(x2.shape[0])
        else:
            strat = ReuseStrategy.by_name(strategy) if strategy else NO_REUSE
            reuse = strat.saves_memory and n >= 2
        key, arena = self._checkout(x2.shape[0], n, strat, reuse)
        self.last_arena = arena
        needs_grad = torch.is_grad_enabled() and (x2.requires_grad or any(p.requires_grad for p in self.parameters()))
        if not needs_grad:
            try:
                return arena.forward(x2).view(shape)
            finally:
                self._return_arena(key, arena)
        lease = _Lease(self, key, arena)
        y = _MoEFunction.apply(x2, self.gate_weight, self.w1, self.w2, lease)
        return y.view(shape)


class StepGraph:
    """One forward + backward of the layer captured as a CUDA graph.

    The whole step — routing kernels, every schedule-DAG op on the compute /
    collective / copy streams with its cross-stream event edges, the gate
    side stream, the deferred weight-gradient GEMMs — is recorded once and
    replayed with a single launch, so launch-bound inner loops (Algorithm 1's
    trials at small batches, small-token steps) cost device time only.
    Inputs are the static buffers `x` / `dy` (copied in by `replay(x, dy)`);
    outputs `y` and `grads` = (dx, dwg, dw1, dw2) are static and overwritten
    by every replay.  The graph owns a private step arena.

    Expert parallel (N > 1, peer memory): the exchanges carry no per-step
    value (flags are raised to 1 and reset by their last waiter, csrc/p2p.cu),
    so the captured flag waits, copy kernels and resets replay unchanged;
    every rank captures and replays its own graph in lock step (collective:
    all ranks construct the StepGraph and call replay the same number of
    times).  The NCCL baseline backend cannot be captured here.
    """

    def __init__(self, layer: "MoELayer", tokens: int, n: int, strategy: ReuseStrategy) -> None:
        if layer.comm.nranks != 1 and getattr(layer.comm, "kind", None) != "p2p":
            raise RuntimeError("StepGraph at N > 1 needs the peer-memory communicator (a2a_backend='p2p')")
        self.layer = layer
        dev, dt = layer.w1.device, layer.w1.dtype
        self.x = torch.zeros(tokens, layer.d_model, device=dev, dtype=dt)
        self.dy = torch.zeros(tokens, layer.d_model, device=dev, dtype=dt)
        reuse = strategy.saves_memory and n >= 2
        key = (tokens, n, strategy.name, bool(reuse), dt, False, layer.wgrad_accumulation)
        self.arena = _Arena(layer, tokens, n, strategy, reuse, dt, False)  # private: never pooled
        self.key = key
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up: first-call host setup happens outside the capture
            self.arena.forward(self.x)
            self.arena.backward(self.x, self.dy)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.y = self.arena.forward(self.x)
            self.grads = self.arena.backward(self.x, self.dy)
        torch.cuda.synchronize()

    def close(self) -> None:
        """Release the graph and its private arena; with peer memory the arena's window is freed
        collectively (every rank closes its StepGraphs in the same order)."""
        self.graph = None
        win, self.arena.win = self.arena.win, None
        if win is not None:
            self.layer.comm.free([win])

    def replay(self, x: torch.Tensor | None = None, dy: torch.Tensor | None = None):
        """Run the captured step on the current stream; returns the static (y, (dx, dwg, dw1, dw2))."""
        if x is not None:
            self.x.copy_(x)
        if dy is not None:
            self.dy.copy_(dy)
        self.graph.replay()
        if self.arena.p2p:
            self.arena.watch(torch.cuda.current_stream().cuda_stream, "MoELayer graph replay")
        return self.y, self.grads
