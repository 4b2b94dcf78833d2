"""`python -m paper_2506_22175_b200.cli` — the reference planner's commands on real hardware.

The reference CLI (`moepipesim {memory,plan,simulate,search,sweep}`,
cli.py:540-573) plans and *simulates* a pipelined MoE layer; this one keeps
its subcommands, flag vocabulary and report schemas (cli.py:614-728) but
drives them with the B200 implementation:

  memory   closed-form Eq. 1-6 report (no GPU)                    cli.py:351-366
  plan     strategy ranking (Eq. 7-8) over a HardwareProfile that   cli.py:369-376
           is *measured* on the GPU (--hardware measured) or read
           from a JSON profile file
  run      the measured counterpart of `simulate`: one real          cli.py:379-401
           forward/backward of MoELayer; makespan, per-stream busy
           time and memory components come from the executed DAG's
           CUDA events (same schema); --out writes the trace
  search   Algorithm 1 over a generated dynamic-B workload with the  cli.py:404-467
           CUDA-event MeasurementAdapter
  sweep    grid of (tokens, n, strategy) measured on the GPU -> CSV  cli.py:477-518
           with the reference's columns

Tokens are routed tokens per GPU (B = T * top_k), as in the
reference.  Errors print one JSON object on stderr; exit status 2 for
usage/config errors, 1 for runtime errors.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import sys
from dataclasses import dataclass, field
from typing import Sequence

from .cost import select_strategy
from .granularity import generate_workload
from .memory import build_report
from .spec import STREAMS, HardwareProfile, ModelSpec, ReuseStrategy, SlowdownTable, micro_batch_size
from .trace import memory_components, us

PRESETS = {  # model presets of the reference (cli.py:46-50) by name, as plain shapes
    "moe-gpt3-s": (768, 3072, 64),
    "moe-gpt3-xl": (2048, 8192, 64),
    "moe-bert-l": (1024, 4096, 64),
}
SWEEP_COLUMNS = ["model_dim", "hidden_dim", "num_experts", "tokens", "partitions", "strategy", "reuse",
                 "micro_batch", "makespan_us", "peak_total_elements", "peak_activations_elements",
                 "peak_buffers_elements", "host_elements"]


class CliUsageError(ValueError):
    """Bad command line."""


class ConfigError(ValueError):
    def __init__(self, message: str, path: str = "") -> None:
        super().__init__(message)
        self.path = path


@dataclass
class Config:
    model_dim: int = 1024
    hidden_dim: int = 4096
    num_experts: int = 64
    num_nodes: int = 8  # the reference default (cli.py); E % num_nodes is validated
    element_bytes: int = 2
    top_k: int = 1
    capacity_factor: float = 1.0
    tokens: int | None = None
    partitions: int | None = None
    adaptive: bool = False
    candidates: tuple = (1, 2, 4, 8, 16)
    trials_per_candidate: int = 1
    min_micro_batch: int = 1
    strategy: str = "none"
    reuse: bool = False
    direction: str = "both"
    hardware: str = "measured"
    seed: int = 0
    out: str | None = None
    trace_format: str = "jsonl"
    workload: dict = field(default_factory=dict)

    @property
    def spec(self) -> ModelSpec:
        return ModelSpec(self.model_dim, self.hidden_dim, self.num_experts, self.num_nodes, self.element_bytes)


_KNOWN = {f for f in Config.__dataclass_fields__} | {"preset"}


def load_config(path: str | None, args: argparse.Namespace) -> Config:
    raw: dict = {}
    if path:
        try:
            with open(path, encoding="utf-8") as fh:
                raw = json.load(fh)
        except (OSError, json.JSONDecodeError) as exc:
            raise ConfigError(f"cannot read config: {exc}", path=path) from None
        if not isinstance(raw, dict):
            raise ConfigError("config must be a JSON object")
        for key in raw:
            if key not in _KNOWN:
                raise ConfigError(f"unknown key {key!r}", path=key)
    flags = {k: v for k, v in vars(args).items() if v is not None and k in _KNOWN}
    raw.update(flags)
    preset = raw.pop("preset", None)
    cfg = Config()
    if preset is not None:
        if preset not in PRESETS:
            raise ConfigError(f"unknown preset {preset!r}", path="preset")
        cfg.model_dim, cfg.hidden_dim, cfg.num_experts = PRESETS[preset]
    n = raw.pop("partitions", None)
    if n is not None:
        if n == "adaptive":
            cfg.adaptive = True
        else:
            try:
                cfg.partitions = int(n)
            except (TypeError, ValueError):
                raise ConfigError(f"n must be an integer or 'adaptive', got {n!r}", path="pipeline.n") from None
    for key, val in raw.items():
        setattr(cfg, key, tuple(val) if key == "candidates" else val)
    if cfg.strategy not in ("none", "s1", "s2", "s3", "s4", "auto"):
        raise ConfigError(f"unknown strategy {cfg.strategy!r}", path="strategy")
    return cfg


def _require(cfg: Config, tokens: bool = False, partitions: bool = False) -> None:
    if tokens and cfg.tokens is None:
        raise ConfigError("batch size required (--batch)", path="batch.tokens")
    if partitions and cfg.partitions is None:
        raise ConfigError("partition count required (--n)", path="pipeline.n")


def _emit(body, out: str | None) -> None:
    text = json.dumps(body, sort_keys=True, indent=2)
    print(text)
    if out:
        with open(out, "w", encoding="utf-8") as fh:
            fh.write(text + "\n")


# ------------------------------------------------------------ hardware
def profile_from_json(d: dict) -> HardwareProfile:
    """HardwareProfile from {"w_comp", "w_comm", "w_mem", "slowdown": [[kind, [others], f], ...] |
    {name: f}, "launch_overhead", "compute_saturation"} (the calibrate / sim_vs_measured format)."""
    sl = d.get("slowdown", {})
    table = (SlowdownTable({(k_, frozenset(s_)): v for k_, s_, v in sl}) if isinstance(sl, list)
             else SlowdownTable.from_factors(**sl))
    return HardwareProfile(float(d["w_comp"]), float(d["w_comm"]), float(d["w_mem"]), table,
                           launch_overhead=float(d.get("launch_overhead", 0.0)),
                           compute_saturation=int(d.get("compute_saturation", 1)))


def profile_to_json(hw: HardwareProfile) -> dict:
    return {"w_comp": hw.w_comp, "w_comm": hw.w_comm, "w_mem": hw.w_mem, "launch_overhead": hw.launch_overhead,
            "compute_saturation": hw.compute_saturation,
            "slowdown": [[k_, sorted(s_), v] for (k_, s_), v in hw.slowdown.entries.items()]}


def _layer(cfg: Config, pipeline=1):
    import torch

    from .layer import MoELayer
    if not torch.cuda.is_available():
        raise RuntimeError("this command runs the CUDA layer; no GPU is visible")
    if cfg.element_bytes != 2:
        raise ConfigError("the measured commands run the bf16 layer (element_bytes 2)", path="model.element_bytes")
    return MoELayer(cfg.model_dim, cfg.hidden_dim, cfg.num_experts, top_k=cfg.top_k,
                    capacity_factor=cfg.capacity_factor, pipeline=pipeline, dtype=torch.bfloat16,
                    candidates=cfg.candidates, trials_per_candidate=cfg.trials_per_candidate,
                    min_micro_batch=cfg.min_micro_batch)


def _tokens_per_rank(cfg: Config, routed: int) -> int:
    return -(-routed // cfg.top_k)


def hardware(cfg: Config, layer=None, routed: int | None = None) -> HardwareProfile:
    if cfg.hardware != "measured":
        try:
            with open(cfg.hardware, encoding="utf-8") as fh:
                return profile_from_json(json.load(fh))
        except (OSError, KeyError, json.JSONDecodeError) as exc:
            raise ConfigError(f"cannot read hardware profile: {exc}", path="hardware") from None
    from .calibrate import measure_profile
    layer = layer or _layer(cfg)
    return measure_profile(layer, tokens=_tokens_per_rank(cfg, routed) if routed else None)


# ------------------------------------------------------------ measured run
def _run_layer(layer, cfg: Config, routed: int, n: int, strategy: ReuseStrategy):
    """One timed forward+backward; returns (fw trace, bw trace, arena)."""
    import torch
    T = _tokens_per_rank(cfg, routed)
    g = torch.Generator(device=layer.w1.device).manual_seed(cfg.seed)
    x = torch.randn(T, cfg.model_dim, device=layer.w1.device, generator=g).bfloat16()
    dy = torch.randn(T, cfg.model_dim, device=layer.w1.device, generator=g).bfloat16()
    layer.record_times = True
    for _ in range(2):  # the first builds the arena
        layer.run_step(x, dy, n, strategy)
    torch.cuda.synchronize()
    arena = layer.last_arena
    fw, bw = arena.traces()
    return fw, bw, arena


def _merged(arena, fw, bw, direction: str):
    """Forward, backward or both (the reference's "both" DAG, backward shifted behind the forward)."""
    from .schedule import build_schedule
    from .spec import NO_REUSE
    from .trace import trace_from_times
    if direction == "forward":
        return fw
    if direction == "backward":
        return bw
    dag = build_schedule(arena.spec, arena.batch, arena.strategy if arena.reuse else NO_REUSE, arena.reuse, "both")
    times = {e.op_id: (e.start, e.end) for e in fw.events}
    shift = fw.makespan
    times.update({e.op_id: (e.start + shift, e.end + shift) for e in bw.events})
    return trace_from_times(dag, times, getattr(arena, "lanes", None))


def _strategy(cfg: Config, layer, routed: int, n: int) -> ReuseStrategy:
    if cfg.strategy == "auto":
        b = micro_batch_size(routed, n)
        return select_strategy(cfg.spec, hardware(cfg, layer, routed), b).strategy
    return ReuseStrategy.by_name(cfg.strategy)


# ------------------------------------------------------------ commands
def cmd_memory(cfg: Config, args) -> int:
    _require(cfg, tokens=True, partitions=True)
    report = build_report(cfg.spec, cfg.tokens, cfg.partitions, reuse=cfg.reuse)
    body = dict(report.to_dict())
    body.update({"model": {"model_dim": cfg.model_dim, "hidden_dim": cfg.hidden_dim,
                           "num_experts": cfg.num_experts, "num_nodes": cfg.num_nodes},
                 "tokens": cfg.tokens, "partitions": cfg.partitions, "reuse": cfg.reuse})
    if args.format in ("json", "both"):
        _emit(body, cfg.out)
    if args.format in ("table", "both"):
        print(report.as_table())
    return 0


def cmd_plan(cfg: Config, args) -> int:
    _require(cfg, tokens=True, partitions=True)
    b = micro_batch_size(cfg.tokens, cfg.partitions)
    hw = hardware(cfg, routed=cfg.tokens)
    body = select_strategy(cfg.spec, hw, b).to_dict()
    body.update({"tokens": cfg.tokens, "partitions": cfg.partitions, "micro_batch": b})
    _emit(body, cfg.out)
    return 0


def cmd_run(cfg: Config, args) -> int:
    _require(cfg, tokens=True, partitions=True)
    from .trace import write_trace
    layer = _layer(cfg)
    strategy = _strategy(cfg, layer, cfg.tokens, cfg.partitions)
    fw, bw, arena = _run_layer(layer, cfg, cfg.tokens, cfg.partitions, strategy)
    trace = _merged(arena, fw, bw, cfg.direction)
    mem = memory_components(trace)
    body = {"strategy": strategy.name, "reuse": bool(arena.reuse), "direction": cfg.direction,
            "tokens": cfg.tokens, "partitions": cfg.partitions, "ops": len(trace.events),
            "makespan_us": us(trace.makespan), "busy_us": {s: us(trace.busy_time(s)) for s in STREAMS},
            "memory": mem.to_dict()}
    print(json.dumps(body, sort_keys=True, indent=2))
    if cfg.out:
        write_trace(trace, cfg.out, cfg.trace_format)
    return 0


def cmd_search(cfg: Config, args) -> int:
    from .calibrate import GpuMeasurementAdapter
    from .granularity import AdaptiveController, TrialBudget
    wl = dict(cfg.workload)
    for key in ("iterations", "b_min", "b_max", "step", "distribution"):
        if getattr(args, key, None) is not None:
            wl[key] = getattr(args, key)
    missing = {"iterations", "b_min", "b_max"} - set(wl)
    if missing:
        raise ConfigError(f"workload needs {sorted(missing)}", path="batch.workload")
    wl.setdefault("seed", cfg.seed)
    try:
        batches = generate_workload(**wl)
    except (TypeError, ValueError) as exc:
        raise ConfigError(str(exc), path="batch.workload") from None
    layer = _layer(cfg)
    strategy = _strategy(cfg, layer, wl["b_max"], max(cfg.candidates))
    adapter = GpuMeasurementAdapter(layer)
    budget = TrialBudget(tuple(cfg.candidates), cfg.trials_per_candidate, adapter, cfg.min_micro_batch)
    ctrl = AdaptiveController(cfg.spec, None, strategy, budget)
    spans: dict = {}
    rows = []
    for it, routed in enumerate(batches):
        before = ctrl.stats.trials
        n = ctrl.adaptive_granularity(routed)
        if (routed, n) not in spans:
            spans[(routed, n)] = adapter(cfg.spec, None, strategy, routed, n)
        rows.append({"iter": it, "B": routed, "n": n, "trials_run": ctrl.stats.trials - before,
                     "makespan_us": us(spans[(routed, n)])})
    if cfg.out:
        with open(cfg.out, "w", encoding="utf-8") as fh:
            fh.write("\n".join(json.dumps(r, sort_keys=True) for r in rows) + "\n")
    _emit({"iterations": len(batches), "strategy": strategy.name, "total_trials": ctrl.stats.trials,
           "total_searches": ctrl.stats.searches, "cache_hit_rate": ctrl.stats.hit_rate,
           "ranges": [{"lo": lo, "hi": hi, "n": n} for lo, hi, n in ctrl.index.ranges]}, None)
    return 0


def cmd_sweep(cfg: Config, args) -> int:
    batches = [int(x) for x in args.batches.split(",")] if args.batches else [cfg.tokens]
    ns = [int(x) for x in args.ns.split(",")] if args.ns else [cfg.partitions]
    names = args.strategies.split(",") if args.strategies else [cfg.strategy]
    if any(b is None for b in batches) or any(n is None for n in ns):
        raise ConfigError("sweep needs --batches/--ns or --batch/--n")
    layer = _layer(cfg)
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=SWEEP_COLUMNS, lineterminator="\n")
    w.writeheader()
    for routed in batches:
        for n in ns:
            for name in names:
                strategy = ReuseStrategy.by_name(name)
                fw, bw, arena = _run_layer(layer, cfg, routed, n, strategy)
                trace = _merged(arena, fw, bw, cfg.direction)
                mem = memory_components(trace)
                w.writerow({"model_dim": cfg.model_dim, "hidden_dim": cfg.hidden_dim,
                            "num_experts": cfg.num_experts, "tokens": routed, "partitions": n,
                            "strategy": strategy.name, "reuse": int(arena.reuse),
                            "micro_batch": micro_batch_size(routed, n), "makespan_us": us(trace.makespan),
                            "peak_total_elements": mem.total, "peak_activations_elements": mem.activations,
                            "peak_buffers_elements": mem.buffers, "host_elements": mem.host})
                layer.last_arena = None
                layer.release_arenas()
    if cfg.out:
        with open(cfg.out, "w", encoding="utf-8", newline="") as fh:
            fh.write(buf.getvalue())
    else:
        sys.stdout.write(buf.getvalue())
    return 0


def cmd_calibrate(cfg: Config, args) -> int:
    """Measure the HardwareProfile on this GPU and print / save it (input of `plan --hardware FILE`)."""
    hw = hardware(Config(**{**cfg.__dict__, "hardware": "measured"}), routed=cfg.tokens)
    _emit(profile_to_json(hw), cfg.out)
    return 0


class _Parser(argparse.ArgumentParser):
    def error(self, message: str) -> None:  # type: ignore[override]
        raise CliUsageError(message)


def _common(p) -> None:
    p.add_argument("--config", help="JSON config file (flat keys of cli.Config)")
    p.add_argument("--preset", choices=sorted(PRESETS))
    p.add_argument("--model-dim", type=int, dest="model_dim")
    p.add_argument("--hidden-dim", type=int, dest="hidden_dim")
    p.add_argument("--num-experts", type=int, dest="num_experts")
    p.add_argument("--num-nodes", type=int, dest="num_nodes")
    p.add_argument("--top-k", type=int, dest="top_k")
    p.add_argument("--capacity-factor", type=float, dest="capacity_factor")
    p.add_argument("--batch", type=int, dest="tokens", help="routed tokens per GPU (B = T * top_k)")
    p.add_argument("--n", dest="partitions", help="partition count, or 'adaptive'")
    p.add_argument("--strategy", choices=["none", "s1", "s2", "s3", "s4", "auto"])
    p.add_argument("--reuse", action="store_true", default=None)
    p.add_argument("--hardware", help="'measured' (calibrate on the GPU) or a JSON profile file")
    p.add_argument("--seed", type=int)
    p.add_argument("--out")
    p.add_argument("--trace-format", choices=["jsonl", "trace-event"], dest="trace_format")
    p.add_argument("--direction", choices=["forward", "backward", "both"])


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="mpm", description="B200 pipelined MoE layer: plan, run and tune")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("memory", help="closed-form memory report")
    _common(p)
    p.add_argument("--format", choices=["json", "table", "both"], default="json")
    p.set_defaults(func=cmd_memory)
    for name, fn, hlp in (("plan", cmd_plan, "strategy ranking over a measured or given profile"),
                          ("run", cmd_run, "one measured forward/backward (reference: simulate)"),
                          ("calibrate", cmd_calibrate, "measure the HardwareProfile on this GPU")):
        p = sub.add_parser(name, help=hlp)
        _common(p)
        p.set_defaults(func=fn)
    p = sub.add_parser("search", help="Algorithm 1 over a workload, GPU-timed")
    _common(p)
    p.add_argument("--iterations", type=int)
    p.add_argument("--b-min", type=int, dest="b_min")
    p.add_argument("--b-max", type=int, dest="b_max")
    p.add_argument("--step", type=int)
    p.add_argument("--distribution", choices=["uniform", "zipf"])
    p.set_defaults(func=cmd_search)
    p = sub.add_parser("sweep", help="measured grid sweep to CSV")
    _common(p)
    p.add_argument("--batches")
    p.add_argument("--ns")
    p.add_argument("--strategies")
    p.set_defaults(func=cmd_sweep)
    return parser


def _error(kind: str, message: str, path: str = "") -> None:
    body = {"error": kind, "message": message}
    if path:
        body["path"] = path
    print(json.dumps(body, sort_keys=True), file=sys.stderr)


def main(argv: Sequence[str] | None = None) -> int:
    try:
        args = build_parser().parse_args(argv)
        cfg = load_config(args.config, args)
        return args.func(cfg, args)
    except CliUsageError as exc:
        _error("usage", str(exc))
        return 2
    except ConfigError as exc:
        _error("config", str(exc), exc.path)
        return 2
    except (ValueError, KeyError, OSError, RuntimeError) as exc:
        _error(type(exc).__name__, str(exc))
        return 1


if __name__ == "__main__":
    sys.exit(main())
