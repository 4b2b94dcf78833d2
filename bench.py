"""Benchmark: MoE layer forward+backward tokens/s (BASELINE.json metric).

Workload (BASELINE.json configs[1], the headline config, per GPU): GPT-MoE
layer d_model=1024, d_ffn=4096, 64 experts top-2, capacity factor 1.0,
16K tokens per GPU, bf16, experts sharded E/N per GPU (N=1: all 64 local).
Synthetic tokens / random-init weights (seeds per SURVEY.md §8d).  One step
= one MoELayer forward + backward (every GEMM, all-to-all, routing and
combine kernel of the path), with the granularity n from Algorithm 1 and
the strategy from `--memory-reuse`.

  python bench.py [--gpus N --steps K --warmup W]          # this framework
  python bench.py --impl reference [...]                   # CPU oracle port

Prints one JSON line (rank 0).  `value` is whole-job tokens/s with inputs
resident in HBM; `e2e` repeats the step through the public API with the
inputs copied host->device from pinned memory inside the timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG = dict(d_model=1024, d_ffn=4096, experts=64, top_k=2, capacity_factor=1.0, tokens_per_gpu=16384)
WORKLOAD = "gpt-moe layer M=1024 H=4096 E=64 top-2 cf=1.0, 16K tokens/GPU, bf16 (BASELINE configs[1])"
METRIC = "MoE layer fwd+bwd tokens/s"


def flops_per_token(M, H, E, k) -> float:
    """Algorithmic fwd+bwd FLOPs per token: 12 k M H (expert FFN) + 6 M E (gate)."""
    return 12.0 * k * M * H + 6.0 * M * E


def choose_peak(peaks: dict, clocks: dict) -> tuple[float, str]:
    """The bf16 denominator for the timed window: the burst figure when the window ran at the maximum
    SM clock with no throttle reason (the kernels saw the clocks the burst GEMM was measured at),
    else the sustained figure (measured back to back for 4 s, power-capped)."""
    sm, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
    throttled = any(r in clocks.get("reasons", []) for r in
                    ("sw_power_cap", "hw_slowdown", "sw_thermal_slowdown", "hw_thermal_slowdown",
                     "hw_power_brake_slowdown"))
    if "bf16_tflops" in peaks and sm and mx and sm >= 0.97 * mx and not throttled:
        return peaks["bf16_tflops"], "MEASURED_PEAKS.json bf16_tflops (burst: timed window at max SM clock, no throttle)"
    if "bf16_tflops_sustained" in peaks:
        return peaks["bf16_tflops_sustained"], "MEASURED_PEAKS.json bf16_tflops_sustained (window below max clock or throttled)"
    return peaks["bf16_tflops"], "MEASURED_PEAKS.json bf16_tflops"


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


# ----------------------------------------------------------------- clocks
REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


_NVML_POLL = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByPciBusId(sys.argv[1])
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
print("ready", flush=True)
while True:
    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    why = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    print(f"{sm},{mx},{why:x},{time.monotonic()!r}", flush=True)
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed region from NVML (the
    counters nvidia-smi reports): by libmpm's native sampler thread every 1 ms (no GIL, so the
    host thread issuing the step cannot starve it), else by a poller process writing to a file,
    else `nvidia-smi -lms 20`.  Samples carry CLOCK_MONOTONIC stamps (time.monotonic); the
    device is found by PCI bus id (CUDA_VISIBLE_DEVICES remapping does not matter)."""

    def __init__(self, index: int) -> None:
        self.index = index
        self.samples: list[tuple[float, float, int, float]] = []
        self._proc = None
        self._thread = None
        self._file = None
        self._native = False

    def _spawn_nvml(self):
        import tempfile

        import torch
        try:
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        except Exception:  # noqa: BLE001
            return None
        self._file = tempfile.NamedTemporaryFile("w+", suffix=".clocks", delete=False)
        proc = subprocess.Popen([sys.executable, "-c", _NVML_POLL, bus], stdout=self._file,
                                stderr=subprocess.DEVNULL, text=True)
        t_end = time.monotonic() + 20.0
        while time.monotonic() < t_end and proc.poll() is None:
            with open(self._file.name) as f:
                if f.readline().strip() == "ready":
                    return proc
            time.sleep(0.01)
        proc.kill()
        return None

    def start(self) -> None:
        # 1st choice: libmpm's native NVML thread (no GIL, in-process: 1 ms cadence under load)
        try:
            if os.environ.get("MPM_CLOCK_NATIVE") == "0":
                raise RuntimeError("native sampler disabled")
            import torch

            from paper_2506_22175_b200 import _lib
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            if _lib.load().mpm_clock_sampler_start(bus.encode(), 1000) == 0:
                self._native = True
                return
        except Exception:  # noqa: BLE001 - fall back to the NVML poller process / nvidia-smi
            pass
        self._proc = self._spawn_nvml()
        if self._proc is not None:
            return
        try:
            self._proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}",
                                           "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                                           "--format=csv,noheader,nounits", "-lms", "20"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return

        def reader():
            for line in self._proc.stdout:
                self._parse(line, time.monotonic())

        self._thread = threading.Thread(target=reader, daemon=True)
        self._thread.start()

    def _parse(self, line: str, now: float) -> None:
        parts = [p.strip() for p in line.split(",")]
        try:
            t = float(parts[3]) if len(parts) > 3 else now
            self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16), t))
        except (ValueError, IndexError):
            pass

    def stop(self, window: tuple[float, float] | None = None) -> dict:
        """Clock summary over the samples taken inside `window` (time.monotonic seconds;
        all samples when none did)."""
        if self._native:
            import ctypes

            from paper_2506_22175_b200 import _lib
            cap = 1 << 16
            buf = (ctypes.c_double * (4 * cap))()
            n = ctypes.c_int(0)
            _lib.load().mpm_clock_sampler_stop(buf, cap, ctypes.byref(n))
            for i in range(n.value):
                self.samples.append((buf[4 * i], buf[4 * i + 1], int(buf[4 * i + 2]), buf[4 * i + 3]))
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
        if self._thread is not None:
            self._thread.join(timeout=2)
        if self._file is not None:
            with open(self._file.name) as f:
                for line in f:
                    self._parse(line, 0.0)
            try:
                os.unlink(self._file.name)
            except OSError:
                pass
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        inside = [s_ for s_ in self.samples if window and window[0] <= s_[3] <= window[1]]
        use = inside or self.samples
        mask = 0
        for _, _, r, _ in use:
            mask |= r
        reasons = [name for bit, name in REASONS.items() if mask & bit and name != "gpu_idle"]
        return {"sm_mhz": statistics.median(s_[0] for s_ in use),
                "sm_max_mhz": max(s_[1] for s_ in use), "reasons": reasons,
                "samples": len(use), "samples_in_timed_region": len(inside)}


# ------------------------------------------------------------ CPU baseline
class CpuOracle:
    """The numpy oracle (fp32) fwd+bwd of the same layer on a bounded token sample."""

    def __init__(self, T_sample: int, seed: int = 0) -> None:
        import numpy as np

        M, H, E = CFG["d_model"], CFG["d_ffn"], CFG["experts"]
        rng = np.random.default_rng(seed)
        self.T = T_sample
        self.x = rng.standard_normal((T_sample, M), dtype=np.float32)
        self.dy = rng.standard_normal((T_sample, M), dtype=np.float32)
        self.wg = (rng.standard_normal((E, M), dtype=np.float32) / np.sqrt(M)).astype(np.float32)
        self.w1 = rng.standard_normal((E, H, M), dtype=np.float32) * np.float32(0.02)
        self.w2 = rng.standard_normal((E, M, H), dtype=np.float32) * np.float32(0.02)

    def step(self) -> float:
        import numpy as np

        from oracle import moe_oracle as O

        t0 = time.perf_counter()
        O.moe_layer([self.x], self.wg, [self.w1], [self.w2], k=CFG["top_k"],
                    capacity_factor=CFG["capacity_factor"], n_chunks=1, dys=[self.dy], dtype=np.float32)
        return time.perf_counter() - t0

    @staticmethod
    def cores() -> int:
        try:
            from threadpoolctl import threadpool_info
            return int(max((i.get("num_threads", 1) for i in threadpool_info()), default=1))
        except Exception:  # pragma: no cover
            return os.cpu_count() or 1

    def sample(self, runs: int) -> str:
        return (f"{self.T} tokens of the same layer (E=64 experts local, top-2, M=1024, H=4096), fp32 numpy "
                f"oracle fwd+bwd, {runs} timed runs, weights generated outside the timed region")


def cpu_oracle_run(T_full: int, budget_s: float = 20.0) -> dict:
    """The CPU baseline at the full per-GPU token count (configs[1]: 16K tokens): one warm-up on a
    512-token sample, then full-size fwd+bwd runs until ~budget_s of CPU work (at least one)."""
    _all_host_threads()
    CpuOracle(512).step()  # warm-up (BLAS threads, allocator)
    orc = CpuOracle(T_full)
    times = [orc.step()]
    while sum(times) < budget_s - times[0] and len(times) < 5:
        times.append(orc.step())
    med = statistics.median(times)
    return {"value": orc.T / med, "unit": "tokens/s", "cores": orc.cores(), "kind": "port",
            "sample": orc.sample(len(times)) + f", median {med:.2f} s", "same_config": True}


def _all_host_threads() -> None:
    """torchrun exports OMP_NUM_THREADS=1; the CPU baseline uses every host core."""
    try:
        import numpy  # noqa: F401  (load the BLAS first: threadpoolctl limits loaded libraries)
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count() or 1)
    except Exception:  # pragma: no cover
        pass


def run_reference(args) -> None:
    """--impl reference: the reference CPU path (the numpy oracle port; the reference package has no
    MoE numerics to run) on the host cores, rank 0 only.  Each step is the full
    configs[1] workload (16K tokens) unless one full step exceeds 8 s on this host, in which case
    every step is a token sample sized to ~6 s (stated in `config.sample_tokens`)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _all_host_threads()
    T = CFG["tokens_per_gpu"]
    CpuOracle(512).step()
    probe = CpuOracle(T).step()
    T_sample = T if probe <= 8.0 else max(512, int(T * 6.0 / probe) // 512 * 512)
    orc = CpuOracle(T_sample)
    for _ in range(max(args.warmup, 1) - 1):
        orc.step()
    times = [orc.step() for _ in range(args.steps)]
    med = statistics.median(times)
    value = orc.T / med
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_tokens": orc.T, "full_step_probe_s": probe},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": orc.cores(), "kind": "port",
                         "sample": orc.sample(len(times)), "same_config": orc.T == T},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def a2a_summary(events, N: int, chunk_rows: list[int], M: int, esz: int, peak_gbs: float = 900.0) -> dict:
    """Per-exchange NVLink traffic of the last timed step from the executor's per-op device times.

    Every chunk exchange (S_i / R_i / BS_i / RC_i / BR_i, pipesim/schedule.py:252-340) moves, per
    rank and direction, chunk_rows[i] (= its experts x its capacity slots) rows of M x esz bytes to /
    from each of the N-1 peers.  `gbs` is those remote bytes over the op's device time (which includes its flag waits,
    i.e. waiting for the slowest peer), against NVLink 5's 900 GB/s per direction."""
    rows = []
    for e in events:
        op = e.op_id
        if not (op[0] in "SR" and not op.startswith("RE")) and not op.startswith(("BS", "BR")):
            continue
        i = int(op.split("_")[-1]) if "_" in op else int(op.lstrip("SRCB"))
        remote = chunk_rows[i] * M * esz * (N - 1)
        dur = e.duration
        rows.append({"op": op, "remote_bytes": remote, "ms": dur * 1e3,
                     "gbs": remote / dur / 1e9 if dur > 0 else None})
    tot_b = sum(r["remote_bytes"] for r in rows)
    tot_s = sum(r["ms"] for r in rows) / 1e3
    mean = tot_b / tot_s / 1e9 if tot_s > 0 else None
    return {"exchanges": rows, "remote_bytes_per_step": tot_b, "busy_ms_per_step": tot_s * 1e3,
            "mean_gbs": mean, "peak_gbs_per_dir": peak_gbs, "frac": mean / peak_gbs if mean else None}


def effective_sm_clock(step, steps: int, dev, interval_us: float = 5.0) -> dict:
    """The SM clock the kernels actually ran at: a separate pass of the same `steps` steps with one
    co-resident warp recording (globaltimer, clock64) pairs (mpm_clock_trace; it sleeps between
    samples, so the pass runs at the headline pass's speed — compare `ms_per_step`).  NVML's SM clock
    reads the maximum during the step while the in-kernel cycle counter shows the power limit pulling
    the clock down within the first step (tools/clock_trace.py, profiles/r2/)."""
    import ctypes

    import torch

    from paper_2506_22175_b200 import _lib
    n = int(steps * 2500 / interval_us) + 2000
    buf = torch.zeros(2 * n, dtype=torch.int64, device=dev)
    side = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()
    time.sleep(0.3)  # the same idle lead-in as the headline pass
    _lib.call("mpm_clock_trace", ctypes.c_void_p(buf.data_ptr()), n, int(interval_us * 1000),
              ctypes.c_void_p(side.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tr = buf.view(n, 2).cpu().tolist()
    gt0 = tr[0][0]
    win = [r for r in tr if 0 < r[0] and r[0] - gt0 <= ms * 1e6]
    if len(win) < 2 or win[-1][0] <= win[0][0]:
        return {"sm_mhz_effective": None, "samples": len(win)}
    mhz = (win[-1][1] - win[0][1]) / (win[-1][0] - win[0][0]) * 1e3
    return {"sm_mhz_effective": round(mhz, 1), "samples": len(win), "ms_per_step": ms / steps,
            "how": "in-kernel clock64 / globaltimer over a separate pass of the same steps (mpm_clock_trace)"}


def max_over_ranks(v: float, dev) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2506_22175_b200 import _lib, ops
    from paper_2506_22175_b200.layer import MoELayer
    from paper_2506_22175_b200.trace import exposed_a2a_fraction

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank; MPM_BENCH_BACKEND=gloo lets ranks share one GPU for a functional
    # check of the N > 1 path (the layer's bytes move over peer memory either way)
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("MPM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    N = world
    M, H, E, k, T = CFG["d_model"], CFG["d_ffn"], CFG["experts"], CFG["top_k"], CFG["tokens_per_gpu"]
    pipeline = "adaptive" if args.n == "adaptive" else int(args.n)
    layer = MoELayer(M, H, E, top_k=k, capacity_factor=CFG["capacity_factor"], pipeline=pipeline,
                     memory_reuse=args.memory_reuse, dtype=torch.bfloat16, device=dev, a2a_backend=args.a2a)
    g = torch.Generator(device="cpu").manual_seed(1000 + rank)
    x_host = torch.randn(T, M, generator=g).bfloat16().pin_memory()
    g = torch.Generator(device="cpu").manual_seed(2000 + rank)
    dy_host = torch.randn(T, M, generator=g).bfloat16().pin_memory()
    x = x_host.to(dev)
    dy = dy_host.to(dev)
    x.requires_grad_(True)

    def step():
        y = layer(x)
        y.backward(dy)
        x.grad = None
        for p in layer.parameters():
            p.grad = None

    n_used, strat, reuse = layer.plan(T)  # runs Algorithm 1 trials on first use
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- timed region (inputs resident): the product path, no per-op instrumentation
    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)  # peak of the timed steps: weights, grads, inputs, one arena
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    k0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    profile = os.environ.get("MPM_PROFILE_TIMED") == "1"  # `ncu --profile-from-start off`: timed steps only
    if profile:
        torch.cuda.profiler.start()
    w0 = time.monotonic()
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    w1 = time.monotonic()
    if profile:
        torch.cuda.profiler.stop()
    kernels = (_lib.launch_count() - k0) // max(args.steps, 1)
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        ms = max_over_ranks(ms, dev)
    time.sleep(0.2)
    clocks = sampler.stop((w0, w1))
    peak_mem = torch.cuda.max_memory_allocated(dev)

    # ---- self-check of the measured configuration (every rank, outside the timed regions):
    # outputs and gradients finite, slot assignment conserves the routed tokens, and (N > 1) the
    # gate gradient all-reduced over peer memory is bit-identical on every rank
    xs = x.detach().clone().requires_grad_(True)
    yc = layer(xs)
    yc.backward(dy)
    grads = [xs.grad, layer.gate_weight.grad, layer.w1.grad, layer.w2.grad]
    st_ = layer.last_arena
    check = {"finite": bool(torch.isfinite(yc).all()) and all(bool(torch.isfinite(t_).all()) for t_ in grads),
             "tokens_conserved": int((st_.slot >= 0).sum()) == int(st_.kept.sum())}
    if world > 1:
        sums = [None] * world
        dist.all_gather_object(sums, layer.gate_weight.grad.double().sum().item())
        check["gate_grad_identical_across_ranks"] = len(set(sums)) == 1
        check["ranks_seen"] = world
    for p_ in layer.parameters():
        p_.grad = None
    if not all(v for k_, v in check.items() if k_ != "ranks_seen"):
        raise RuntimeError(f"bench self-check failed: {check}")

    # ---- clock pass: the effective SM clock of the same steps (in-kernel cycle counter)
    eff_clock = effective_sm_clock(step, args.steps, dev)

    # ---- second timed pass with per-op CUDA events on every schedule op (device timestamps on
    # each op's own stream): the GEMM time behind `roofline` and the step breakdown.  Separate
    # from the headline pass because the events themselves cost a few percent of the step.
    layer.last_arena = None
    layer.release_arenas()
    layer.record_times = True
    step()  # builds the timing arena outside the timed pass
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record()
    for _ in range(max(3, min(args.steps, 10))):
        step()
    pe1.record()
    torch.cuda.synchronize()
    ms_instrumented = pe0.elapsed_time(pe1) / max(3, min(args.steps, 10))
    arena = layer.last_arena
    layer.record_times = False

    # roofline of the dominant kernel class (tcgen05 grouped expert GEMMs): per-op
    # device timestamps of the last timed step (ops C_i, RE_i, G2_i, G1_i)
    fw, bw = arena.traces()
    # device time covered by GEMM ops: the union of their intervals per trace (with two compute lanes
    # the GEMMs of consecutive chunks overlap, so a plain sum would double count)
    from paper_2506_22175_b200.trace import _union
    gemm_s = sum(sum(b_ - a_ for a_, b_ in _union([(e.start, e.end) for e in tr.events
                                                    if e.op_id.startswith(("C", "RE", "G2_", "G1_"))]))
                 for tr in (fw, bw)) + arena.wgrad_seconds()
    from paper_2506_22175_b200.trace import exposed_time
    exposed_ms = (exposed_time(fw) + exposed_time(bw)) * 1e3  # collective busy time not under compute
    a2a = None
    if N > 1:
        g_ = arena.g
        rows_ = [g_.chunk(i).ne * g_.chunk(i).cs for i in range(g_.n)]
        a2a = a2a_summary([e for tr in (fw, bw) for e in tr.events], N, rows_, M, 2)
        a2a.update(backend=getattr(layer.comm, "kind", "none"), ranks=N,
                   exposed_ms_per_step=exposed_ms,
                   # the byte counts above are capacity volumes; with the compacted expert side only
                   # the routed rows (this share of the capacity slots) cross NVLink
                   compacted=bool(getattr(arena, "compact", False)),
                   routed_fraction=float(arena.kept.sum()) / (g_.E * g_.C))
    # device-time breakdown of the last timed step (per schedule op; the rest is routing /
    # combine / gate kernels and launch gaps on the compute stream)
    breakdown = {"forward_span_ms": fw.makespan * 1e3, "backward_span_ms": bw.makespan * 1e3,
                 "ops_ms": {e.op_id: round(e.duration * 1e3, 4) for tr in (fw, bw) for e in tr.events
                            if e.duration > 0},
                 "deferred_wgrad_ms": arena.wgrad_seconds() * 1e3, "phases_ms": arena.phase_ms()}
    C = ops.capacity(T, k, E, CFG["capacity_factor"])
    rows = E * C  # expert rows computed per GPU (capacity-padded slots, all chunks)
    gemm_flops = 2.0 * rows * M * H * (2 + 4 + (1 if reuse and strat.restore_middle.value == "recompute" else 0))
    # algorithmic (routed-token) flops inside those GEMMs: 12 k M H per token
    alg_gemm_flops = 12.0 * k * M * H * T
    peaks = load_peaks()
    peak_tf, peak_source = choose_peak(peaks, clocks)
    # the tensor pipe's own rate at the clock the kernels ran at: 148 SMs x 8192 dense bf16 FLOP per
    # SM clock (tcgen05 M=128 N=256 K=16 per 128 cycles per SM) x the in-kernel effective SM clock —
    # what ncu's tensor-pipe-active % measures against (the cuBLAS burst figure was itself taken at
    # an unknown, power-limited clock, so it does not scale with the clock ratio)
    f_eff = eff_clock.get("sm_mhz_effective")
    # the clock reading only describes the headline pass when the traced pass ran at its speed
    eff_ms = eff_clock.get("ms_per_step")
    if f_eff and eff_ms and abs(eff_ms / ms - 1.0) > 0.1:
        eff_clock["rejected"] = (f"traced pass {eff_ms:.3f} ms/step vs headline {ms:.3f}: the tracer "
                                 "disturbed the steps, so its clock does not describe the headline pass")
        f_eff = None
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_eff = sms * 8192 * f_eff * 1e6 / 1e12 if f_eff else None
    if "fallback" in peaks:
        peak_source = "fallback (B200_PROFILING.md)"
    achieved = alg_gemm_flops / gemm_s / 1e12 if gemm_s > 0 else None
    traffic = None
    prof = ROOT / "profiles" / "gemm_traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_step")
    # the GEMMs' algorithmic DRAM bytes (every operand and output touched once, bf16, 1-bit masks):
    # expert weights read by fc1/fc2/both dgrads and written by both wgrads, activations/gradients
    # of width M and H six times each, the ReLU mask written once and read once
    R = (E // N) * N * ops.capacity(T, k, E, CFG["capacity_factor"])  # expert-side rows per GPU
    alg_gemm_bytes = 6 * (E // N) * M * H * 2 + 6 * R * M * 2 + 6 * R * H * 2 + 2 * R * H // 8

    value = N * T / (ms / 1e3)

    # ---- e2e through the public API with host buffers: every step copies its inputs x and dy
    # from pinned host memory and reads its outputs y and dx back into pinned host memory
    # (double-buffered on two copy streams so step i's transfers overlap steps i-1 / i+1, the
    # way an input pipeline prefetches and a host consumer drains); the weight gradients stay
    # on the device for the optimizer.  Both directions cross PCIe inside the timed region.
    h2d = 2 * T * M * 2  # x and dy, bf16
    d2h = 2 * T * M * 2  # y and dx, bf16
    h2d_stream, d2h_stream = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    xbuf = [torch.empty(T, M, device=dev, dtype=torch.bfloat16) for _ in range(2)]
    dybuf = [torch.empty(T, M, device=dev, dtype=torch.bfloat16) for _ in range(2)]
    y_host = [torch.empty(T, M, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
    dx_host = [torch.empty(T, M, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
    outs: list = [None, None]
    ready = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    produced = [torch.cuda.Event() for _ in range(2)]
    drained = [torch.cuda.Event() for _ in range(2)]
    compute = torch.cuda.current_stream()

    def prefetch(i):
        b = i % 2
        h2d_stream.wait_event(consumed[b])
        with torch.cuda.stream(h2d_stream):
            xbuf[b].copy_(x_host, non_blocking=True)
            dybuf[b].copy_(dy_host, non_blocking=True)
        ready[b].record(h2d_stream)

    def e2e_step(i):
        b = i % 2
        compute.wait_event(ready[b])
        compute.wait_event(drained[b])  # y_host / dx_host[b] free again
        xd = xbuf[b].detach().requires_grad_(True)
        y = layer(xd)
        y.backward(dybuf[b])
        consumed[b].record(compute)
        produced[b].record(compute)
        outs[b] = (y, xd.grad)  # keep alive until the read-back below is stream-ordered
        d2h_stream.wait_event(produced[b])
        with torch.cuda.stream(d2h_stream):
            y_host[b].copy_(y.detach(), non_blocking=True)
            dx_host[b].copy_(xd.grad, non_blocking=True)
        drained[b].record(d2h_stream)
        for p in layer.parameters():
            p.grad = None

    for b in range(2):
        consumed[b].record(compute)
        drained[b].record(compute)
    prefetch(0)
    for i in range(2):  # warm-up
        prefetch(i + 1)
        e2e_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(2, 2 + args.steps):
        prefetch(i + 1)
        e2e_step(i)
    compute.wait_stream(d2h_stream)  # the last step's outputs are on the host before the clock stops
    e1.record()
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1) / args.steps
    if world > 1:
        ms_e2e = max_over_ranks(ms_e2e, dev)
    assert bool(torch.isfinite(y_host[(1 + args.steps) % 2].float()).all())
    e2e = {"value": N * T / (ms_e2e / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
           "note": "x, dy pinned host -> device and y, dx device -> pinned host every step, overlapped "
                   "with the neighbouring steps on two copy streams; weight gradients stay on the device"}

    # ---- memory reuse (the metric's peak-memory part): arena bytes and step time
    # at n=4 without reuse and with each strategy, next to the paper's Eq. 6 bound
    memory = None
    if not args.no_memory_sweep:
        from paper_2506_22175_b200.memory import mem_saving_ratio
        from paper_2506_22175_b200.spec import ModelSpec
        sweep = {}
        n_mem = 4
        import gc
        for name in ("none", "s4", "s3", "s2", "s1"):
            layer.last_arena = None  # every arena of the previous strategy is dropped before measuring
            layer.release_arenas()
            gc.collect()
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats(dev)
            base = torch.cuda.memory_allocated(dev)

            def mstep():
                y = layer(x, n=n_mem, strategy=None if name == "none" else name)
                y.backward(dy)
                x.grad = None
                for p in layer.parameters():
                    p.grad = None

            mstep()
            torch.cuda.synchronize()
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record()
            for _ in range(3):
                mstep()
            m1.record()
            torch.cuda.synchronize()
            sweep[name] = {"arena_bytes": layer.last_arena.device_bytes,
                           "arena_by_category": dict(layer.last_arena.bytes_by_category),
                           "peak_allocated_bytes": torch.cuda.max_memory_allocated(dev) - base,
                           "ms_per_step": m0.elapsed_time(m1) / 3}
        layer.release_arenas()
        E_tokens = ops.capacity(T, k, E, CFG["capacity_factor"]) * E
        spec = ModelSpec(M, H, E, N, 2)
        memory = {"n": n_mem, "strategies": sweep,
                  "act_buf_saving_vs_none": {
                      s_: 1 - (v["arena_by_category"].get("activations", 0) + v["arena_by_category"].get("buffers", 0))
                      / (sweep["none"]["arena_by_category"]["activations"] + sweep["none"]["arena_by_category"]["buffers"])
                      for s_, v in sweep.items() if s_ != "none"},
                  "phi_eq6": mem_saving_ratio(spec, E_tokens, n_mem),
                  "note": "arena = activations + gradient scratch + routing (allocated-capacity convention); "
                          "at N=1 dispatch/combine are identities so T_DI/T_DO alias T_I/T_O"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_run(T)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": N, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "tokens_per_gpu": T, "experts_per_gpu": E // N,
                       "pipeline_n": n_used, "memory_reuse": strat.name if reuse else "none",
                       "parallelism": f"ep{N}", "a2a": getattr(layer.comm, "kind", "none") if N > 1 else "identity (N=1)",
                       "l2": "no flush; per-step working set (1 GiB expert weights + 0.5 GiB activations) >> 126 MB L2"},
            "roofline": {"bound": "tensor", "kernel": "tcgen05 grouped expert GEMM (all fc1/fc2 fwd/dgrad/wgrad)",
                         "measured_in": "instrumented timed pass (per-op CUDA events, last step)",
                         "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": (achieved / peak_tf) if achieved else None, "traffic": traffic,
                         "peak_source": peak_source,
                         "frac_vs_burst": achieved / peaks["bf16_tflops"] if achieved and peaks.get("bf16_tflops") else None,
                         "frac_vs_sustained": achieved / peaks["bf16_tflops_sustained"]
                         if achieved and peaks.get("bf16_tflops_sustained") else None,
                         # tensor-pipe rate at the measured effective SM clock (clocks.effective)
                         "peak_at_effective_clock": peak_eff,
                         "frac_vs_effective_clock_peak": achieved / peak_eff if achieved and peak_eff else None,
                         "algorithmic_flops_per_step": alg_gemm_flops,
                         "executed_flops_per_step": gemm_flops, "gemm_ms_per_step": gemm_s * 1e3,
                         "hbm_view": {"algorithmic_bytes_per_step": alg_gemm_bytes,
                                      "achieved_gbs": alg_gemm_bytes / gemm_s / 1e9 if gemm_s > 0 else None,
                                      "peak_gbs": peaks.get("hbm_gbs"),
                                      "frac": (alg_gemm_bytes / gemm_s / 1e9 / peaks["hbm_gbs"])
                                      if gemm_s > 0 and peaks.get("hbm_gbs") else None}},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": kernels * args.steps,
            "gpu_launches_per_step": kernels, "clocks": {**clocks, "effective": eff_clock},
            "peak_memory_bytes": peak_mem, "arena_bytes": arena.device_bytes, "memory_reuse_sweep": memory,
            "step_breakdown": breakdown, "ms_per_step_instrumented": ms_instrumented,
            "exposed_a2a_frac": exposed_ms / ms_instrumented if ms_instrumented > 0 else None,
            "exposed_a2a_frac_fwd_bwd_dag": [exposed_a2a_fraction(fw), exposed_a2a_fraction(bw)],
            "a2a": a2a, "self_check": check,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pipeline-n", "--n", dest="n", default="adaptive",
                    help="granularity n or 'adaptive' (under torchrun spell it --pipeline-n: torchrun reads --n as its own)")
    ap.add_argument("--memory-reuse", default="none")
    ap.add_argument("--a2a", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 exchange backend: peer-memory copy kernels (default) or NCCL send/recv (baseline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-memory-sweep", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
