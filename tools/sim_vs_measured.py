"""Calibrated HardwareProfile + simulated-vs-measured makespan.

  measure  (GPU box)   python tools/sim_vs_measured.py measure --out F.json
      measures the HardwareProfile of the cfg2 layer on the device
      (calibrate.measure_profile: w_comp, w_mem, the comp/mem interference
      factors; w_comm at N=1 is "infinite" — the exchanges are identities),
      then runs the real pipelined layer for a set of (n, strategy) and
      records the measured forward / backward DAG makespans and per-op
      durations (runtime.PipelineExecutor CUDA events, reference trace
      schema).
  simulate (here, needs /root/reference)
           python tools/sim_vs_measured.py simulate --in F.json --out G.json
      feeds that profile to the UNMODIFIED reference simulator
      (moepipesim.simulate, pipesim/engine.py:114-322) on the same
      schedules and writes predicted vs measured makespans side by side —
      the check of the cost model's inputs the paper's Eq. 8 relies on.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CASES = [(1, "none"), (2, "none"), (4, "none"), (8, "none"), (2, "s4"), (4, "s4"), (8, "s4"), (4, "s3"),
         (4, "s1"), (4, "s2")]
M, H, E, K, T = 1024, 4096, 64, 2, 16384


def measure(args) -> None:
    import torch

    from paper_2506_22175_b200.calibrate import measure_profile
    from paper_2506_22175_b200.layer import MoELayer
    from paper_2506_22175_b200.spec import NO_REUSE, ReuseStrategy
    from paper_2506_22175_b200.trace import event_rows

    dev = torch.device("cuda", 0)
    # one compute stream, as the reference's model has (the second compute lane is a B200 addition)
    layer = MoELayer(M, H, E, top_k=K, capacity_factor=1.0, pipeline=1, dtype=torch.bfloat16, device=dev,
                     compute_lanes=1)
    hw = measure_profile(layer, tokens=T)
    out = {"layer": {"M": M, "H": H, "E": E, "k": K, "T": T, "N": 1},
           "profile": {"w_comp": hw.w_comp, "w_comm": hw.w_comm, "w_mem": hw.w_mem,
                       "launch_overhead": hw.launch_overhead, "compute_saturation": hw.compute_saturation,
                       "slowdown": [[k_, sorted(s_), v] for (k_, s_), v in hw.slowdown.entries.items()]},
           "cases": []}
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(T, M, device=dev, generator=g, dtype=torch.bfloat16)
    dy = torch.randn(T, M, device=dev, generator=g, dtype=torch.bfloat16)
    layer.record_times = True
    for n, strategy in CASES:
        strat = NO_REUSE if strategy == "none" else ReuseStrategy.by_name(strategy)
        for _ in range(3):
            layer.run_step(x, dy, n, strat)
        torch.cuda.synchronize()
        a = layer.last_arena
        fw, bw = a.traces()
        out["cases"].append({"n": n, "strategy": strategy, "reuse": a.reuse,
                             "measured_fwd_makespan": fw.makespan, "measured_bwd_makespan": bw.makespan,
                             "deferred_wgrad_s": a.wgrad_seconds(), "phases_ms": a.phase_ms(),
                             "fwd_events": event_rows(fw), "bwd_events": event_rows(bw)})
        layer.last_arena = None
        layer.release_arenas()
        print(n, strategy, fw.makespan, bw.makespan, flush=True)
    Path(args.out).write_text(json.dumps(out, indent=1))


def simulate(args) -> None:
    import os
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.path.insert(0, "/root/reference/pkg/src")
    import moepipesim as R
    from moepipesim.pipesim import build_schedule, simulate as sim

    data = json.loads(Path(args.inp).read_text())
    p = data["profile"]
    table = R.SlowdownTable({(k_, frozenset(s_)): v for k_, s_, v in p["slowdown"]})
    hw = R.HardwareProfile(p["w_comp"], min(p["w_comm"], 1e300), p["w_mem"], table,
                           launch_overhead=p["launch_overhead"], compute_saturation=p["compute_saturation"])
    lay = data["layer"]
    spec = R.ModelSpec(lay["M"], lay["H"], lay["E"], lay["N"], 2)
    C = -(-lay["T"] * lay["k"] // lay["E"])
    rows = []
    for case in data["cases"]:
        n, strategy = case["n"], case["strategy"]
        strat = R.NO_REUSE if strategy == "none" else getattr(R, strategy.upper())
        reuse = bool(case["reuse"])
        batch = R.BatchSpec(lay["E"] * C, n)
        pred = {}
        for direction in ("forward", "backward"):
            dag = build_schedule(spec, batch, strat if reuse else R.NO_REUSE, reuse, direction)
            pred[direction] = sim(dag, hw).makespan
        meas_bw = case["measured_bwd_makespan"] + case["deferred_wgrad_s"]
        rows.append({"n": n, "strategy": strategy, "reuse": reuse,
                     "sim_fwd_ms": pred["forward"] * 1e3, "measured_fwd_ms": case["measured_fwd_makespan"] * 1e3,
                     "sim_bwd_ms": pred["backward"] * 1e3, "measured_bwd_ms": meas_bw * 1e3,
                     "fwd_ratio": case["measured_fwd_makespan"] / pred["forward"],
                     "bwd_ratio": meas_bw / pred["backward"]})
    out = {"profile": p, "note": "reference simulator (moepipesim 0.1.0, unmodified) fed the B200-measured "
                                 "profile; measured = CUDA-event makespan of the executed DAG (backward "
                                 "includes the deferred weight-gradient GEMMs, which the reference folds "
                                 "into G1/G2)", "rows": rows}
    Path(args.out).write_text(json.dumps(out, indent=1))
    print(f"{'n':>3} {'strategy':>8} {'sim fwd':>9} {'meas fwd':>9} {'sim bwd':>9} {'meas bwd':>9}")
    for r in rows:
        print(f"{r['n']:>3} {r['strategy']:>8} {r['sim_fwd_ms']:9.3f} {r['measured_fwd_ms']:9.3f} "
              f"{r['sim_bwd_ms']:9.3f} {r['measured_bwd_ms']:9.3f}")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["measure", "simulate"])
    ap.add_argument("--out", required=True)
    ap.add_argument("--in", dest="inp")
    args = ap.parse_args()
    measure(args) if args.mode == "measure" else simulate(args)


if __name__ == "__main__":
    main()
