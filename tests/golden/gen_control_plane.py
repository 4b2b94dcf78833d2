"""Generate tests/golden/control_plane.json from the UNMODIFIED reference.

Run in the build container (the reference is mounted read-only there):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_control_plane.py

The fixture freezes the reference's outputs (moepipesim 0.1.0,
/root/reference/pkg) for the control-plane functions on the hot path
(SURVEY.md §8a rows a1-a13), so the GPU box — where /root/reference does
not exist — checks this framework's planner against the same numbers.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.append("/root/reference/pkg/src")

import moepipesim as R  # noqa: E402
from moepipesim.pipesim import simulate  # noqa: E402
from moepipesim.pipesim.engine import memory_components  # noqa: E402

OUT = Path(__file__).with_name("control_plane.json")

SPECS = {
    "gpt3_s": (768, 3072, 64, 8), "gpt3_xl": (2048, 8192, 64, 8), "bert_l": (1024, 4096, 64, 8),
    "tiny": (16, 64, 8, 8), "cfg1": (256, 1024, 4, 1), "cfg2": (1024, 4096, 64, 8), "cfg3": (2048, 8192, 32, 8),
    "cfg4": (4096, 16384, 64, 8), "cfg5": (1024, 4096, 128, 8),
}
PROFILES = {
    "flat": dict(w_comp=1e12, w_comm=1e10, w_mem=1e10, compute_saturation=1),
    "interfering": dict(w_comp=1e12, w_comm=1e10, w_mem=1e10, compute_saturation=1,
                        slowdown=dict(mu_comp=0.8, mu_all=0.6, sigma_comm=0.9, eta_all=0.7)),
    "b200_guess": dict(w_comp=7.0e14, w_comm=4.57e11, w_mem=2.75e10, compute_saturation=1024,
                       launch_overhead=5e-6, slowdown=dict(mu_comp=0.8, mu_all=0.6, eta_all=0.7)),
    "comm_bound": dict(w_comp=1e12, w_comm=1e9, w_mem=2e9,
                       slowdown=dict(mu_comp=0.9, mu_all=0.5, eta_all=0.5)),
    "copy_cheap": dict(w_comp=1e12, w_comm=5e11, w_mem=1e12,
                       slowdown=dict(mu_comp=0.9, mu_all=0.85, eta_all=0.9)),
}


def profile(d):
    d = dict(d)
    slow = d.pop("slowdown", {})
    return R.HardwareProfile(d.pop("w_comp"), d.pop("w_comm"), d.pop("w_mem"),
                             R.SlowdownTable.from_factors(**slow), **d)


def dag_dict(dag):
    return {
        "ops": {k: [v.kind, v.partition, v.stream, v.work, v.tokens, list(v.deps)] for k, v in dag.ops.items()},
        "issue_order": {k: list(v) for k, v in dag.issue_order.items()},
        "pools": {k: [v.category, v.capacity, v.slot_elements] for k, v in dag.pools.items()},
        "slots": [[s.pool, s.acquire, list(s.releases)] for s in dag.slots],
        "host_slices": [[h.elements, h.producer] for h in dag.host_slices],
    }


def main():
    out = {"reference": "moepipesim " + R.__version__ if hasattr(R, "__version__") else "moepipesim 0.1.0"}
    out["partition_sizes"] = [[B, n, R.BatchSpec(B, n).partition_sizes(), R.micro_batch_size(B, n)]
                              for B, n in [(2048, 2), (32768, 4), (65536, 16), (10, 3), (1, 1), (999, 7),
                                           (512, 4), (80, 3)]]
    out["strategies"] = {s.name: [s.restore_dispatched_input.value, s.restore_middle.value, list(s.q_fw),
                                  list(s.q_bw), s.comm_slowdown_mode, s.copy_slowdown_mode]
                         for s in R.STRATEGIES.values()}
    mem = []
    for name, (M, H, E, N) in SPECS.items():
        spec = R.ModelSpec(M, H, E, N)
        for B in (1, 4096, 8192, 16384, 32768, 65536, 1310720):
            for n in (1, 2, 4, 8, 16):
                if n > B:
                    continue
                for reuse in ([False, True] if n >= 2 else [False]):
                    rep = R.build_report(spec, B, n, reuse)
                    mem.append([name, B, n, reuse, rep.model_states, rep.activations, rep.buffers,
                                rep.saving_ratio])
    out["memory"] = mem
    cost = []
    for pname, pd in PROFILES.items():
        hw = profile(pd)
        for sname in ("tiny", "gpt3_s", "cfg2", "cfg4"):
            spec = R.ModelSpec(*SPECS[sname])
            for b in (1, 512, 1024, 2048, 8192, 16384):
                sel = R.select_strategy(spec, hw, b)
                costs = {k: [fw.t_comp, fw.t_comm, fw.t_mem, bw.t_comp, bw.t_comm, bw.t_mem]
                         for k, (fw, bw) in sel.costs.items()}
                cost.append([pname, sname, b, sel.strategy.name, costs])
    out["cost"] = cost
    dags = []
    for sname in ("tiny", "cfg1"):
        spec = R.ModelSpec(*SPECS[sname])
        for n in (1, 2, 3, 4):
            for strat in ("none", "s1", "s2", "s3", "s4"):
                s = R.ReuseStrategy.by_name(strat)
                reuse = s.saves_memory and n >= 2
                if strat != "none" and not reuse:
                    continue
                for direction in ("forward", "backward", "both"):
                    B = 64 * n + (n - 1)  # uneven partitions
                    dag = R.build_schedule(spec, R.BatchSpec(B, n), s, reuse, direction)
                    entry = {"spec": sname, "tokens": B, "n": n, "strategy": strat, "reuse": reuse,
                             "direction": direction, "dag": dag_dict(dag)}
                    tr = simulate(dag, profile(PROFILES["interfering"]))
                    entry["times"] = {e.op_id: [e.start, e.end] for e in tr.events}
                    mc = memory_components(tr)
                    entry["memory_components"] = [mc.model_states, mc.activations, mc.buffers, mc.host]
                    dags.append(entry)
    out["schedules"] = dags

    # Algorithm 1 against a deterministic, non-monotone stub adapter
    def stub(spec, hw, strategy, tokens, partitions):
        best = 1 if tokens < 3000 else 2 if tokens < 9000 else 4 if tokens < 20000 else 8
        if tokens in (12288, 25600):  # contradicting votes exercise the clip path
            best = 2
        return abs(partitions - best) + partitions * 1e-6 + (tokens % 7) * 1e-9

    spec = R.ModelSpec(*SPECS["gpt3_s"])
    alg = []
    for seed, dist_name in ((7, "uniform"), (11, "zipf")):
        work = R.generate_workload(seed, 400, 1024, 32768, dist_name, step=512)
        budget = R.TrialBudget(candidates=(1, 2, 4, 8, 16), adapter=stub, min_micro_batch=256)
        ctrl = R.AdaptiveController(spec, profile(PROFILES["flat"]), R.NO_REUSE, budget)
        decisions = [ctrl.adaptive_granularity(b) for b in work]
        st = ctrl.stats
        alg.append({"seed": seed, "distribution": dist_name, "workload": work, "decisions": decisions,
                    "ranges": ctrl.index.ranges, "conflicts": ctrl.index.conflicts,
                    "stats": [st.calls, st.cache_hits, st.range_hits, st.searches, st.trials],
                    "max_probes": ctrl.index.max_probes_per_find})
    out["algorithm1"] = alg
    out["workloads"] = [[seed, it, lo, hi, d, step, R.generate_workload(seed, it, lo, hi, d, step=step)]
                        for seed, it, lo, hi, d, step in [(9, 50, 1024, 4096, "uniform", 512),
                                                          (3, 200, 1024, 32768, "zipf", 1024),
                                                          (0, 5, 7, 7, "uniform", 1)]]
    OUT.write_text(json.dumps(out, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
