"""Control-plane parity: this framework's planner vs the reference (moepipesim).

Two pins, both runnable without a GPU:
  * golden constants copied from the reference's own tests (cited inline);
  * tests/golden/control_plane.json, generated from the unmodified
    reference by tests/golden/gen_control_plane.py (schedules, pools, slot
    wiring, memory closed forms, cost model / strategy choice, Algorithm 1
    decisions and ranges, workload sequences, simulated-trace memory).
"""

import json
import math
from pathlib import Path

import pytest

import paper_2506_22175_b200 as P
from paper_2506_22175_b200 import trace as TR
from paper_2506_22175_b200.cost import _PREFERENCE
from paper_2506_22175_b200.granularity import AdaptiveController, GranularityIndex, TrialBudget
from paper_2506_22175_b200.schedule import ScheduleError, build_schedule

FIX = json.loads((Path(__file__).parent / "golden" / "control_plane.json").read_text())
SPECS = {
    "gpt3_s": (768, 3072, 64, 8), "gpt3_xl": (2048, 8192, 64, 8), "bert_l": (1024, 4096, 64, 8),
    "tiny": (16, 64, 8, 8), "cfg1": (256, 1024, 4, 1), "cfg2": (1024, 4096, 64, 8), "cfg3": (2048, 8192, 32, 8),
    "cfg4": (4096, 16384, 64, 8), "cfg5": (1024, 4096, 128, 8),
}
GPT3_S = P.ModelSpec(768, 3072, 64, 8)
GPT3_XL = P.ModelSpec(2048, 8192, 64, 8)
BERT_L = P.ModelSpec(1024, 4096, 64, 8)


def profile(d):
    d = dict(d)
    slow = d.pop("slowdown", {})
    return P.HardwareProfile(d.pop("w_comp"), d.pop("w_comm"), d.pop("w_mem"),
                             P.SlowdownTable.from_factors(**slow), **d)


PROFILES = {
    "flat": dict(w_comp=1e12, w_comm=1e10, w_mem=1e10, compute_saturation=1),
    "interfering": dict(w_comp=1e12, w_comm=1e10, w_mem=1e10, compute_saturation=1,
                        slowdown=dict(mu_comp=0.8, mu_all=0.6, sigma_comm=0.9, eta_all=0.7)),
    "b200_guess": dict(w_comp=7.0e14, w_comm=4.57e11, w_mem=2.75e10, compute_saturation=1024,
                       launch_overhead=5e-6, slowdown=dict(mu_comp=0.8, mu_all=0.6, eta_all=0.7)),
    "comm_bound": dict(w_comp=1e12, w_comm=1e9, w_mem=2e9, slowdown=dict(mu_comp=0.9, mu_all=0.5, eta_all=0.5)),
    "copy_cheap": dict(w_comp=1e12, w_comm=5e11, w_mem=1e12,
                       slowdown=dict(mu_comp=0.9, mu_all=0.85, eta_all=0.9)),
}


# ------------------------------------------------------------ golden constants (reference tests)
def test_micro_batch_examples():  # test_core.py:26-29
    assert P.micro_batch_size(8192, 4) == 2048
    assert P.micro_batch_size(10, 3) == 4
    assert P.micro_batch_size(4096, 1) == 4096
    for bad in [(10, 11), (10, 0), (0, 1), (5, -1)]:
        with pytest.raises(P.InvalidPartitioningError):
            P.micro_batch_size(*bad)


def test_table2_q_vectors():  # test_core.py:71-83
    expected = {"none": ((2, 2, 0), (4, 2, 0)), "s1": ((2, 2, 5), (4, 2, 5)), "s2": ((2, 2, 4), (4, 3, 4)),
                "s3": ((2, 2, 1), (5, 2, 1)), "s4": ((2, 2, 0), (5, 3, 0))}
    assert set(P.STRATEGIES) == set(expected)
    for name, (fw, bw) in expected.items():
        s = P.ReuseStrategy.by_name(name)
        assert (s.q_fw, s.q_bw) == (fw, bw)
    with pytest.raises(KeyError):
        P.ReuseStrategy.by_name("s9")


def test_memory_frozen_values():  # test_memmodel.py:27-98
    assert P.mem_model_states(GPT3_S) == 19_070_976
    assert P.mem_model_states(GPT3_XL) == 134_742_016
    assert P.mem_activations_baseline(GPT3_S, 4096) == 25_165_824
    assert P.mem_buffers_baseline(GPT3_S, 4096) == 15_728_640
    assert P.mem_buffers_baseline(BERT_L, 8192) == 41_943_040
    assert P.mem_pipeline(GPT3_S, 16384) == (100_663_296, 100_663_296)
    assert P.mem_reuse_savings(GPT3_S, 4096, 2) == 6_291_456
    assert P.mem_reuse_savings(GPT3_S, 16384, 8) == 62_914_560
    assert P.mem_reuse_savings(GPT3_XL, 8192, 4) == 67_108_864
    assert P.mem_saving_ratio(GPT3_S, 16384, 8) == pytest.approx(0.5709, abs=1e-4)
    with pytest.raises(P.ReuseNotApplicableError):
        P.mem_reuse_savings(GPT3_S, 4096, 1)


def test_cost_frozen_values():  # test_costmodel.py:22-43
    v = P.base_volumes(GPT3_S, 1024)
    assert (v.v_comp, v.v_comm, v.v_mem) == (2_415_919_104, 786_432, 786_432)
    hw = P.HardwareProfile(1e12, 1e10, 2e10, P.SlowdownTable.from_factors(mu_comp=0.9), compute_saturation=1024)
    cb = P.stage_cost(GPT3_S, hw, 1024, P.NO_REUSE, "forward")
    assert cb.t_comp == pytest.approx(4.831838208e-3, rel=1e-12)
    assert cb.t_comm == pytest.approx(1.7476266666666666e-4, rel=1e-12)
    assert cb.t_mem == 0.0
    assert _PREFERENCE == ("s4", "s3", "s2", "s1")


def test_slowdown_resolution():  # test_core.py:116-127
    t = P.SlowdownTable.from_factors(mu_comp=0.9, mu_all=0.6, eta_all=0.7)
    assert t.factor("comm", set()) == 1.0
    assert t.factor("comm", {"comp"}) == 0.9
    assert t.factor("comm", {"comp", "mem"}) == 0.6
    assert t.factor("comm", {"mem"}) == 1.0
    assert t.factor("mem", {"comp", "comm"}) == 0.7
    assert P.SlowdownTable.from_factors(mu_comp=0.9, mu_mem=0.8).factor("comm", {"comp", "mem"}) == 0.8
    for bad in [{("comm", frozenset()): 0.9}, {("comm", frozenset({"comp"})): 0.0},
                {("bogus", frozenset({"comp"})): 0.5}, {("comm", frozenset({"comm"})): 0.5}]:
        with pytest.raises(ValueError):
            P.SlowdownTable(bad)


def test_issue_orders():  # test_schedule.py:36-41,107,121-127
    spec = P.ModelSpec(16, 64, 8, 8)
    dag = build_schedule(spec, P.BatchSpec(256, 4), P.NO_REUSE, False, "forward")
    assert dag.issue_order["collective"] == ("S0", "S1", "R0", "S2", "R1", "S3", "R2", "R3")
    s4 = build_schedule(spec, P.BatchSpec(128, 2), P.S4, True, "backward")
    assert s4.issue_order["collective"][:4] == ("BS0", "RC0", "BS1", "RC1")
    s1 = build_schedule(spec, P.BatchSpec(192, 3), P.S1, True, "both")
    assert s1.issue_order["copy"] == ("Ddi0", "Dm0", "Ddi1", "Dm1", "Ddi2", "Dm2",
                                      "Hdi0", "Hm0", "Hdi1", "Hm1", "Hdi2", "Hm2")
    with pytest.raises(P.ReuseNotApplicableError):
        build_schedule(spec, P.BatchSpec(64, 1), P.S1, True)
    with pytest.raises(ValueError):
        build_schedule(spec, P.BatchSpec(64, 2), P.NO_REUSE, True)


def test_conflict_clipping_golden():  # test_autotune.py:127-139
    votes = {2048: 2, 6144: 4, 10240: 2}
    stub = lambda spec, hw, s, B, n: abs(n - votes[B]) + n * 1e-6
    ctrl = AdaptiveController(P.ModelSpec(64, 256, 8, 8), None, P.NO_REUSE,
                              TrialBudget(candidates=(1, 2, 4), adapter=stub))
    for b in (2048, 6144, 10240):
        ctrl.adaptive_granularity(b)
    assert ctrl.index.conflicts == 1
    assert ctrl.index.ranges == [(2048, 6143, 2), (6144, 6144, 4)]
    assert ctrl.index.cache[10240] == 2
    ctrl.index.check_integrity()


def test_find_is_logarithmic_and_index_roundtrips():  # test_autotune.py:59-66
    idx = GranularityIndex()
    for i in range(1024):
        idx.insert(10 * i, 10 * i + 5, i + 1)
    for b in (0, 3, 5000, 5121, 10237, 7):
        idx.find(b)
    assert idx.max_probes_per_find <= math.ceil(math.log2(len(idx))) + 1
    idx.cache[3] = 1
    again = GranularityIndex.from_json(idx.to_json())
    assert again.ranges == idx.ranges and again.cache == idx.cache


# --------------------------------------------------------------------- fixture parity
def test_partition_sizes_fixture():
    for B, n, sizes, mb in FIX["partition_sizes"]:
        assert P.BatchSpec(B, n).partition_sizes() == sizes
        assert P.micro_batch_size(B, n) == mb


def test_strategy_table_fixture():
    for name, (tdi, tm, qf, qb, cm, ym) in FIX["strategies"].items():
        s = P.STRATEGIES[name]
        assert [s.restore_dispatched_input.value, s.restore_middle.value, list(s.q_fw), list(s.q_bw),
                s.comm_slowdown_mode, s.copy_slowdown_mode] == [tdi, tm, qf, qb, cm, ym]


def test_memory_fixture():
    for name, B, n, reuse, ms, act, buf, ratio in FIX["memory"]:
        rep = P.build_report(P.ModelSpec(*SPECS[name]), B, n, reuse)
        assert (rep.model_states, rep.activations, rep.buffers) == (ms, act, buf)
        assert rep.saving_ratio == ratio


def test_cost_and_selection_fixture():
    for pname, sname, b, chosen, costs in FIX["cost"]:
        sel = P.select_strategy(P.ModelSpec(*SPECS[sname]), profile(PROFILES[pname]), b)
        assert sel.strategy.name == chosen
        for k, vals in costs.items():
            fw, bw = sel.costs[k]
            assert [fw.t_comp, fw.t_comm, fw.t_mem, bw.t_comp, bw.t_comm, bw.t_mem] == pytest.approx(vals, rel=1e-15)


def _dag_dict(dag):
    return {
        "ops": {k: [v.kind, v.partition, v.stream, v.work, v.tokens, list(v.deps)] for k, v in dag.ops.items()},
        "issue_order": {k: list(v) for k, v in dag.issue_order.items()},
        "pools": {k: [v.category, v.capacity, v.slot_elements] for k, v in dag.pools.items()},
        "slots": [[s.pool, s.acquire, list(s.releases)] for s in dag.slots],
        "host_slices": [[h.elements, h.producer] for h in dag.host_slices],
    }


def test_schedule_fixture_and_trace_accounting():
    assert len(FIX["schedules"]) > 50
    for e in FIX["schedules"]:
        spec = P.ModelSpec(*SPECS[e["spec"]])
        dag = build_schedule(spec, P.BatchSpec(e["tokens"], e["n"]), P.STRATEGIES[e["strategy"]], e["reuse"],
                             e["direction"])
        mine = _dag_dict(dag)
        ref = e["dag"]
        assert mine["ops"] == ref["ops"]
        assert mine["issue_order"] == ref["issue_order"]
        assert mine["pools"] == ref["pools"]
        assert sorted(map(json.dumps, mine["slots"])) == sorted(map(json.dumps, ref["slots"]))
        assert mine["host_slices"] == ref["host_slices"]
        # the reference simulator's timeline through this framework's trace tooling
        tr = TR.trace_from_times(dag, {k: tuple(v) for k, v in e["times"].items()})
        TR.replay_validate(tr, slack=1e-12)
        mc = TR.memory_components(tr)
        assert [mc.model_states, mc.activations, mc.buffers, mc.host] == e["memory_components"]


def test_algorithm1_fixture():
    def stub(spec, hw, strategy, tokens, partitions):
        best = 1 if tokens < 3000 else 2 if tokens < 9000 else 4 if tokens < 20000 else 8
        if tokens in (12288, 25600):
            best = 2
        return abs(partitions - best) + partitions * 1e-6 + (tokens % 7) * 1e-9

    for e in FIX["algorithm1"]:
        assert P.generate_workload(e["seed"], 400, 1024, 32768, e["distribution"], step=512) == e["workload"]
        budget = TrialBudget(candidates=(1, 2, 4, 8, 16), adapter=stub, min_micro_batch=256)
        ctrl = AdaptiveController(GPT3_S, None, P.NO_REUSE, budget)
        assert [ctrl.adaptive_granularity(b) for b in e["workload"]] == e["decisions"]
        assert [list(r) for r in ctrl.index.ranges] == e["ranges"]
        assert ctrl.index.conflicts == e["conflicts"]
        st = ctrl.stats
        assert [st.calls, st.cache_hits, st.range_hits, st.searches, st.trials] == e["stats"]
        assert ctrl.index.max_probes_per_find == e["max_probes"]


def test_workload_fixture():
    for seed, it, lo, hi, d, step, seq in FIX["workloads"]:
        assert P.generate_workload(seed, it, lo, hi, d, step=step) == seq


def test_trace_validator_catches_early_slot_reuse():
    spec = P.ModelSpec(16, 64, 8, 8)
    dag = build_schedule(spec, P.BatchSpec(256, 4), P.S4, True, "forward")
    # serial timeline in the executor's host issue order -> valid
    from paper_2506_22175_b200.runtime import Pool, plan_dag
    pools = {k: Pool(k, p.capacity, [None] * p.capacity) for k, p in dag.pools.items()
             if k not in ("t_i", "t_o")}
    t, times = 0.0, {}
    for o, _, _ in plan_dag(dag, pools):
        times[o] = (t, t + 1.0)
        t += 1.0
    TR.replay_validate(TR.trace_from_times(dag, times))
    # S2 (third t_di acquisition, capacity 2) starts before C0 released slot 0
    bad = dict(times)
    bad["S2"] = (times["C0"][0] - 0.5, times["C0"][0] - 0.25)
    with pytest.raises(TR.TraceInvariantError):
        TR.replay_validate(TR.trace_from_times(dag, bad))


# --------------------------------------------------------------- direct reference comparison
@pytest.mark.reference
def test_direct_against_reference_randomized(moepipesim):
    import random

    R = moepipesim
    rng = random.Random(20261017)
    for _ in range(300):
        M, H = rng.randint(1, 4096), rng.randint(1, 16384)
        N = rng.choice([1, 2, 4, 8])
        E = N * rng.randint(1, 16)
        spec_p, spec_r = P.ModelSpec(M, H, E, N), R.ModelSpec(M, H, E, N)
        B = rng.randint(1, 1 << 20)
        n = rng.choice([2, 3, 4, 8, 16])
        if n <= B:
            assert P.build_report(spec_p, B, n, True).to_dict() == R.build_report(spec_r, B, n, True).to_dict()
        b = rng.randint(1, 1 << 16)
        kw = dict(mu_comp=rng.uniform(0.3, 1), mu_all=rng.uniform(0.3, 1), eta_all=rng.uniform(0.3, 1),
                  sigma_comm=rng.uniform(0.5, 1))
        w = [rng.uniform(1e9, 1e15), rng.uniform(1e8, 1e12), rng.uniform(1e8, 1e11)]
        sat = rng.randint(1, 4096)
        hp = P.HardwareProfile(*w, P.SlowdownTable.from_factors(**kw), compute_saturation=sat)
        hr = R.HardwareProfile(*w, R.SlowdownTable.from_factors(**kw), compute_saturation=sat)
        assert P.select_strategy(spec_p, hp, b).to_dict() == R.select_strategy(spec_r, hr, b).to_dict()
