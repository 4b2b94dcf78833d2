"""bench.py helpers that run without a GPU: the algorithmic FLOP count behind `roofline`,
and the clock sampler's parsing / timed-window summary behind `clocks`."""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_flops_per_token_matches_survey():
    # cfg2 = 101,056,512 FLOPs per token (12 k M H + 6 M E)
    assert bench.flops_per_token(1024, 4096, 64, 2) == 101_056_512
    assert bench.flops_per_token(256, 1024, 4, 1) == 3_151_872  # cfg1


def test_clock_summary_uses_the_timed_window_and_names_reasons():
    s = bench.ClockSampler(0)
    # nvidia-smi style (hex reasons, no stamp) and poller/native style (stamped) lines
    s._parse("1965, 1965, 0x0000000000000000", 0.5)
    s._parse("1965,1965,4,1.0", 0.0)          # sw_power_cap inside the window
    s._parse("1500,1965,0,1.1", 0.0)
    s._parse("900,1965,20,5.0", 0.0)          # sw_thermal_slowdown, after the window
    s._parse("garbage line", 0.0)
    out = s.stop((0.9, 2.0))
    assert out["samples_in_timed_region"] == 2
    assert out["sm_mhz"] == (1965 + 1500) / 2 and out["sm_max_mhz"] == 1965
    assert out["reasons"] == ["sw_power_cap"]
    # no sample inside the window: all samples summarise the run
    s2 = bench.ClockSampler(0)
    s2._parse("1965,1965,40,3.0", 0.0)
    out2 = s2.stop((0.0, 1.0))
    assert out2["samples_in_timed_region"] == 0 and out2["reasons"] == ["hw_thermal_slowdown"]
    assert bench.ClockSampler(0).stop()["reasons"] == ["unavailable"]


def test_a2a_summary_counts_remote_bytes_per_exchange():
    from types import SimpleNamespace as NS
    ev = [NS(op_id="S0", duration=1e-5), NS(op_id="C0", duration=5e-5), NS(op_id="R0", duration=2e-5),
          NS(op_id="BS_1", duration=1e-5), NS(op_id="RE_1", duration=1e-5), NS(op_id="BR_1", duration=1e-5),
          NS(op_id="RC_0", duration=1e-5)]
    out = bench.a2a_summary(ev, N=8, chunk_rows=[8 * 256, 8 * 256], M=1024, esz=2)
    ops_ = [r["op"] for r in out["exchanges"]]
    assert ops_ == ["S0", "R0", "BS_1", "BR_1", "RC_0"]  # no compute / recompute ops
    per = 256 * 8 * 1024 * 2 * 7  # c_i x E_loc x M x bytes x (N-1) peers
    assert all(r["remote_bytes"] == per for r in out["exchanges"])
    assert abs(out["exchanges"][0]["gbs"] - per / 1e-5 / 1e9) < 1e-6
    assert out["remote_bytes_per_step"] == 5 * per and out["peak_gbs_per_dir"] == 900.0


def test_peak_choice_follows_the_timed_window_clocks():
    peaks = {"bf16_tflops": 1669.6, "bf16_tflops_sustained": 1397.2}
    assert bench.choose_peak(peaks, {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": []})[0] == 1669.6
    assert bench.choose_peak(peaks, {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": ["sw_power_cap"]})[0] == 1397.2
    assert bench.choose_peak(peaks, {"sm_mhz": 1500, "sm_max_mhz": 1965, "reasons": []})[0] == 1397.2
