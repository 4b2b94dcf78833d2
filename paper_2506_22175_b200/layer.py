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
                   compute / copy streams (schedule.build_schedule executed
                   by runtime.PipelineExecutor)
  compute stream   weighted combine of T_O -> y
Backward mirrors it (combine_bwd -> BS/RC/Hdi/Hm/RE/G2/G1/BR -> gather +
gate backward), then one all-reduce of the replicated gate's gradient
(data parallel).

The granularity n comes from Algorithm 1 (granularity.AdaptiveController)
with a CUDA-event-timed measurement of this very layer; the reuse strategy
from cost.select_strategy over a HardwareProfile measured on the device
(calibrate.py) when memory_reuse="auto".
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist
from torch import nn

from . import _lib, ops
from .comm import ExpertComm
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


@dataclass(frozen=True)
class Geometry:
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
    def sizes(self) -> list[int]:
        return balanced_split(self.C, self.n)

    @property
    def starts(self) -> list[int]:
        out, acc = [], 0
        for s in self.sizes:
            out.append(acc)
            acc += s
        return out

    def rows(self, i: int) -> int:
        """Rows per local expert in chunk i (all sources)."""
        return self.N * self.sizes[i]

    @property
    def max_rows(self) -> int:
        return self.N * max(self.sizes)


def _region(buf: torch.Tensor, g: Geometry, i: int) -> torch.Tensor:
    """Chunk i of a chunk-major [E*C, W] buffer as [E, c_i, W]."""
    s, c = g.starts[i], g.sizes[i]
    return buf[g.E * s: g.E * (s + c)].view(g.E, c, buf.shape[-1])


def _expert_view(flat: torch.Tensor, g: Geometry, i: int, width: int) -> torch.Tensor:
    """[E_loc, N*c_i, width] view of a ring buffer (or an aliased region)."""
    R = g.rows(i)
    return flat.reshape(-1)[: g.e_loc * R * width].view(g.e_loc, R, width)


class _Step:
    """Device state and schedule execution of one forward (+ backward) call."""

    def __init__(self, layer: "MoELayer", x: torch.Tensor, n: int, strategy: ReuseStrategy,
                 reuse: bool, record_times: bool = False) -> None:
        self.layer = layer
        self.x = x
        T, M = x.shape
        comm = layer.comm
        C = ops.capacity(T, layer.top_k, layer.num_experts, layer.capacity_factor)
        if C < 1:
            raise InvalidPartitioningError(f"capacity {C} < 1 for T={T}")
        if not 1 <= n <= C:
            raise InvalidPartitioningError(f"pipeline granularity n={n} must be in [1, C={C}]")
        self.g = Geometry(T, M, layer.d_hidden, layer.num_experts, comm.nranks, comm.rank, layer.top_k, C, n)
        self.strategy = strategy
        self.reuse = reuse and n >= 2 and strategy.saves_memory
        self.record_times = record_times
        self.spec = ModelSpec(M, layer.d_hidden, layer.num_experts, comm.nranks,
                              element_bytes=x.element_size())
        self.batch = BatchSpec(self.g.E * C, n)
        self.fw_trace = self.bw_trace = None
        self.alloc_bytes = 0

    # --------------------------------------------------------------- buffers
    def _empty(self, *shape, dtype=None) -> torch.Tensor:
        t = torch.empty(*shape, device=self.x.device, dtype=dtype or self.x.dtype)
        self.alloc_bytes += t.numel() * t.element_size()
        return t

    def _ring(self, name: str, cap: int, width: int) -> Pool:
        g = self.g
        bufs = [self._empty(g.e_loc * g.max_rows * width) for _ in range(cap)]
        return Pool(name, cap, bufs)

    def _streams(self) -> dict[str, torch.cuda.Stream]:
        lay = self.layer
        return {COMPUTE_STREAM: torch.cuda.current_stream(), COLLECTIVE_STREAM: lay._stream("collective"),
                COPY_STREAM: lay._stream("copy")}

    # --------------------------------------------------------------- forward
    def forward(self) -> torch.Tensor:
        lay, g, x = self.layer, self.g, self.x
        compute = torch.cuda.current_stream()
        origin = None
        if self.record_times:
            origin = torch.cuda.Event(enable_timing=True)
            origin.record(compute)
        self.routing = ops.compute_routing(x, lay.gate_weight, g.k, g.C, lay.renorm)
        self.t_i = self._empty(g.E * g.C, g.M)
        ops.permute(x, self.routing, g.n, self.t_i)
        self.t_o = self._empty(g.E * g.C, g.M)

        dag = build_schedule(self.spec, self.batch, self.strategy if self.reuse else NO_REUSE,
                             reuse_enabled=self.reuse, direction=FORWARD)
        self.fw_dag = dag
        pools = {}
        if g.N == 1:
            pools["t_di"] = Pool("t_di", 1, alias=lambda i: _region(self.t_i, g, i))
            pools["t_do"] = Pool("t_do", 1, alias=lambda i: _region(self.t_o, g, i))
        else:
            pools["t_di"] = self._ring("t_di", dag.pools["t_di"].capacity, g.M)
            pools["t_do"] = self._ring("t_do", dag.pools["t_do"].capacity, g.M)
        pools["t_m"] = self._ring("t_m", dag.pools["t_m"].capacity, g.H)
        self.pools = pools
        self.host_di = self.host_m = None
        if self.reuse and self.strategy.restore_dispatched_input is RestoreMethod.OFFLOAD and g.N > 1:
            self.host_di = [lay._pinned(("di", i), g.e_loc * g.rows(i) * g.M, x.dtype) for i in range(g.n)]
        if self.reuse and self.strategy.restore_middle is RestoreMethod.OFFLOAD:
            self.host_m = [lay._pinned(("m", i), g.e_loc * g.rows(i) * g.H, x.dtype) for i in range(g.n)]

        pre = torch.cuda.Event()
        pre.record(compute)
        ex = PipelineExecutor(dag, self._streams(), self._impl, pools, self.record_times)
        ex.run(after=pre)
        ex.join(compute)
        self.fw_exec = ex
        y = ops.combine(self.t_o, self.routing, g.n, g.T)
        if self.record_times:
            self.fw_origin = origin
        return y

    # -------------------------------------------------------------- backward
    def backward(self, dy: torch.Tensor):
        lay, g, x = self.layer, self.g, self.x
        compute = torch.cuda.current_stream()
        origin = None
        if self.record_times:
            origin = torch.cuda.Event(enable_timing=True)
            origin.record(compute)
        self.g_o = self._empty(g.E * g.C, g.M)
        dprob = ops.combine_bwd(dy, self.t_o, self.routing, g.n, self.g_o)
        self.g_i = self._empty(g.E * g.C, g.M)

        dag = build_schedule(self.spec, self.batch, self.strategy if self.reuse else NO_REUSE,
                             reuse_enabled=self.reuse, direction=BACKWARD)
        self.bw_dag = dag
        pools = self.pools
        for p in pools.values():
            p.reset_ring()
        if g.N == 1:
            pools["g_do"] = Pool("g_do", 1, alias=lambda i: _region(self.g_o, g, i))
            pools["g_di"] = Pool("g_di", 1, alias=lambda i: _region(self.g_i, g, i))
        else:
            pools["g_do"] = self._ring("g_do", dag.pools["g_do"].capacity, g.M)
            pools["g_di"] = self._ring("g_di", dag.pools["g_di"].capacity, g.M)
        pools["g_m"] = self._ring("g_m", dag.pools["g_m"].capacity, g.H)

        w1, w2 = lay.w1, lay.w2
        self.dw1 = torch.empty_like(w1)
        self.dw2 = torch.empty_like(w2)
        if g.n > 1 and w1.dtype != torch.float32:
            self.acc1 = self._empty(*w1.shape, dtype=torch.float32)
            self.acc2 = self._empty(*w2.shape, dtype=torch.float32)
        else:
            self.acc1 = self.acc2 = None

        pre = torch.cuda.Event()
        pre.record(compute)
        ex = PipelineExecutor(dag, self._streams(), self._impl, pools, self.record_times)
        ex.run(after=pre)
        ex.join(compute)
        self.bw_exec = ex

        dlogits = ops.gate_bwd_logits(self.routing, dprob, lay.renorm)
        dx = ops.gather_bwd(self.g_i, self.routing, dlogits, lay.gate_weight, g.n, g.T)
        dwg = ops.gate_wgrad(dlogits, x)
        if g.N > 1:
            dist.all_reduce(dwg, group=lay.group)
        if self.record_times:
            self.bw_origin = origin
        dw1, dw2 = self.dw1, self.dw2
        self._release()
        return dx, dwg, dw1, dw2

    def _release(self) -> None:
        """Drop the step's device buffers (every stream was joined into compute)."""
        for name in ("t_i", "t_o", "g_o", "g_i", "acc1", "acc2", "dw1", "dw2", "host_di", "host_m"):
            setattr(self, name, None)
        for p in self.pools.values():
            p.buffers = []
            p.by_partition = {}
            p.alias = None

    # ------------------------------------------------------- op realisations
    def _wgrad_epilogue(self, i: int, dw: torch.Tensor, acc: torch.Tensor | None):
        """(c, epilogue, aux) of chunk i's weight-gradient GEMM (fp32 accumulation over chunks)."""
        n = self.g.n
        if n == 1:
            return dw, _lib.EPI_NONE, None
        if acc is None:  # fp32 weights: accumulate in place
            return dw, (_lib.EPI_STORE_F32 if i == 0 else _lib.EPI_ACCUM_F32), None
        if i == 0:
            return acc, _lib.EPI_STORE_F32, None
        if i < n - 1:
            return acc, _lib.EPI_ACCUM_F32, None
        return dw, _lib.EPI_ADD_AUX_F32, acc

    def _impl(self, op_id: str, ex: PipelineExecutor) -> None:
        g, lay = self.g, self.layer
        node = ex.dag.ops[op_id]
        i = node.partition
        c_i = g.sizes[i]
        M, H, E_loc = g.M, g.H, g.e_loc
        comm = lay.comm
        view = lambda pool, w: _expert_view(ex.buffer(pool, i), g, i, w)
        if op_id.startswith("RC") or (op_id[0] == "S"):
            # dispatch / re-dispatch T_I chunk -> T_DI (identity at N == 1)
            if g.N > 1:
                comm.a2a(_lib.A2A_DISPATCH, _region(self.t_i, g, i), view("t_di", M), E_loc, c_i, M)
        elif op_id[0] == "C":
            t_di, t_m = view("t_di", M), view("t_m", H)
            ops.gemm(t_di, lay.w1, t_m, epilogue=_lib.EPI_RELU)
            ops.gemm(t_m, lay.w2, view("t_do", M))
        elif op_id[0] == "R" and not op_id.startswith("RE"):
            if g.N > 1:
                comm.a2a(_lib.A2A_COMBINE, view("t_do", M), _region(self.t_o, g, i), E_loc, c_i, M)
        elif op_id.startswith("Ddi"):
            if self.host_di is not None:
                ops.copy_async(self.host_di[i], view("t_di", M).reshape(-1))
        elif op_id.startswith("Dm"):
            ops.copy_async(self.host_m[i], view("t_m", H).reshape(-1))
        elif op_id.startswith("BS"):
            if g.N > 1:
                comm.a2a(_lib.A2A_DISPATCH, _region(self.g_o, g, i), view("g_do", M), E_loc, c_i, M)
        elif op_id.startswith("Hdi"):
            if self.host_di is not None:
                ops.copy_async(view("t_di", M).reshape(-1), self.host_di[i])
        elif op_id.startswith("Hm"):
            ops.copy_async(view("t_m", H).reshape(-1), self.host_m[i])
        elif op_id.startswith("RE"):
            ops.gemm(view("t_di", M), lay.w1, view("t_m", H), epilogue=_lib.EPI_RELU)
        elif op_id.startswith("G2_"):
            g_do, t_m, g_m = view("g_do", M), view("t_m", H), view("g_m", H)
            ops.gemm(g_do, lay.w2, g_m, b_mn_major=True, epilogue=_lib.EPI_DRELU, aux=t_m)
            c, epi, aux = self._wgrad_epilogue(i, self.dw2, self.acc2)
            ops.gemm(g_do, t_m, c, a_mn_major=True, b_mn_major=True, epilogue=epi, aux=aux)
        elif op_id.startswith("G1_"):
            g_m, t_di, g_di = view("g_m", H), view("t_di", M), view("g_di", M)
            ops.gemm(g_m, lay.w1, g_di, b_mn_major=True)
            c, epi, aux = self._wgrad_epilogue(i, self.dw1, self.acc1)
            ops.gemm(g_m, t_di, c, a_mn_major=True, b_mn_major=True, epilogue=epi, aux=aux)
        elif op_id.startswith("BR"):
            if g.N > 1:
                comm.a2a(_lib.A2A_COMBINE, view("g_di", M), _region(self.g_i, g, i), E_loc, c_i, M)
        else:  # pragma: no cover - build_schedule emits nothing else
            raise RuntimeError(f"no realisation for op {op_id}")

    def traces(self):
        """Measured (forward, backward) ScheduleTraces (synchronises)."""
        from .trace import trace_from_times
        fw = trace_from_times(self.fw_dag, self.fw_exec.times(self.fw_origin))
        bw = trace_from_times(self.bw_dag, self.bw_exec.times(self.bw_origin)) if hasattr(self, "bw_exec") else None
        return fw, bw


class _MoEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, gate_weight, w1, w2, step: _Step):
        y = step.forward()
        ctx.step = step
        return y

    @staticmethod
    def backward(ctx, dy):
        step = ctx.step
        dx, dwg, dw1, dw2 = step.backward(dy.contiguous())
        ctx.step = None
        return dx, dwg, dw1, dw2, None


class MoELayer(nn.Module):
    """Pipelined expert-parallel MoE FFN layer (tcgen05 experts, NCCL all-to-all).

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
    """

    def __init__(self, d_model: int, d_hidden: int, num_experts: int, top_k: int = 1,
                 capacity_factor: float = 1.0, pipeline=True, memory_reuse=False, renorm: bool = True,
                 group=None, dtype: torch.dtype = torch.bfloat16, device=None,
                 candidates=(1, 2, 4, 8, 16), trials_per_candidate: int = 1, min_micro_batch: int = 1,
                 hw_profile=None, seed: int = 0) -> None:
        super().__init__()
        self.d_model, self.d_hidden, self.num_experts = d_model, d_hidden, num_experts
        self.top_k, self.capacity_factor, self.renorm = top_k, capacity_factor, renorm
        self.group = group
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.comm = ExpertComm(group, device)
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
        self._streams: dict[str, torch.cuda.Stream] = {}
        self._pinned_cache: dict = {}
        self.record_times = False
        self.last_step: _Step | None = None

    # ------------------------------------------------------------ plumbing
    def reset_parameters(self, seed: int = 0) -> None:
        """x-independent synthetic init: W_g ~ N(0, 1/M) (seed 7), W1/W2 ~ N(0, 0.02^2) (seed 11+rank)."""
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

    # ------------------------------------------------------------ planning
    def capacity(self, tokens: int) -> int:
        return ops.capacity(tokens, self.top_k, self.num_experts, self.capacity_factor)

    def model_spec(self, element_bytes: int | None = None) -> ModelSpec:
        return ModelSpec(self.d_model, self.d_hidden, self.num_experts, self.comm.nranks,
                         element_bytes or self.w1.element_size())

    def hardware_profile(self):
        if self.hw_profile is None:
            from .calibrate import measure_profile
            self.hw_profile = measure_profile(self)
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
            strategy = select_strategy(self.model_spec(), self.hardware_profile(),
                                       math.ceil(self.num_experts * C / n)).strategy
        elif self.memory_reuse not in ("none", "auto"):
            strategy = ReuseStrategy.by_name(self.memory_reuse)
        return n, strategy, strategy.saves_memory and n >= 2

    def _adaptive_n(self, tokens: int) -> int:
        if self._controller is None:
            from .granularity import AdaptiveController, TrialBudget
            from .calibrate import GpuMeasurementAdapter
            budget = TrialBudget(self.candidates, self.trials_per_candidate, GpuMeasurementAdapter(self),
                                 self.min_micro_batch)
            strategy = NO_REUSE if self.memory_reuse in ("none", "auto") else ReuseStrategy.by_name(self.memory_reuse)
            self._controller = AdaptiveController(self.model_spec(), None, strategy, budget)
        routed = tokens * self.top_k
        n = self._controller.adaptive_granularity(routed)
        return max(1, min(n, self.capacity(tokens)))

    # ------------------------------------------------------------ forward
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
        step = _Step(self, x2, n, strat, reuse, record_times=self.record_times)
        self.last_step = step if self.record_times else None
        y = _MoEFunction.apply(x2, self.gate_weight, self.w1, self.w2, step)
        return y.view(shape)
