"""CLI (`python -m paper_2506_22175_b200.cli`): the reference planner's commands and report schemas
(cli.py:540-728).  CPU tests: memory / plan outputs equal the unmodified reference CLI's for the same
config (when /root/reference is mounted) and validate against its JSON schemas; error paths print
machine-readable JSON with the reference's exit codes.  GPU test: run / sweep / search end to end."""

import csv
import io
import json
import os
import sys
from pathlib import Path

import pytest

from paper_2506_22175_b200 import cli

REF = Path("/root/reference/pkg/src")


def _ref_cli():
    if not REF.exists():
        pytest.skip("reference not mounted")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    from moepipesim import cli as rcli
    return rcli


def _run(capsys, argv):
    rc = cli.main(argv)
    out = capsys.readouterr()
    return rc, out.out, out.err


@pytest.mark.parametrize("preset,batch,n,reuse", [("moe-gpt3-s", 16384, 8, True), ("moe-bert-l", 8192, 4, False),
                                                  ("moe-gpt3-xl", 4096, 1, False)])
def test_memory_matches_reference_cli(capsys, preset, batch, n, reuse):
    argv = ["memory", "--preset", preset, "--batch", str(batch), "--n", str(n)] + (["--reuse"] if reuse else [])
    rc, out, _ = _run(capsys, argv)
    assert rc == 0
    ours = json.loads(out)
    rcli = _ref_cli()
    assert rcli.main(argv) == 0
    ref = json.loads(capsys.readouterr().out)
    assert ours == ref
    import jsonschema
    jsonschema.validate(ours, rcli.REPORT_SCHEMAS["memory"])


def test_plan_with_profile_file_matches_reference(tmp_path, capsys):
    prof = {"w_comp": 6.1e14, "w_comm": 4.5e11, "w_mem": 2.8e10, "launch_overhead": 5e-6, "compute_saturation": 16000,
            "slowdown": [["comp", ["mem"], 0.86], ["mem", ["comp"], 0.99], ["comm", ["comp"], 0.8]]}
    pf = tmp_path / "hw.json"
    pf.write_text(json.dumps(prof))
    rc, out, _ = _run(capsys, ["plan", "--preset", "moe-bert-l", "--batch", "32768", "--n", "4",
                               "--hardware", str(pf)])
    assert rc == 0
    ours = json.loads(out)
    rcli = _ref_cli()
    cfg = {"model": {"preset": "moe-bert-l"}, "hardware": {
        "w_comp": prof["w_comp"], "w_comm": prof["w_comm"], "w_mem": prof["w_mem"],
        "launch_overhead": prof["launch_overhead"], "compute_saturation": prof["compute_saturation"],
        "slowdown": {"sigma_mem": 0.86, "eta_comp": 0.99, "mu_comp": 0.8}}}
    cf = tmp_path / "ref.json"
    cf.write_text(json.dumps(cfg))
    assert rcli.main(["plan", "--config", str(cf), "--batch", "32768", "--n", "4"]) == 0
    ref = json.loads(capsys.readouterr().out)
    assert ours["chosen"] == ref["chosen"]
    for name in ("none", "s1", "s2", "s3", "s4"):
        assert ours["strategies"][name]["total"] == pytest.approx(ref["strategies"][name]["total"], rel=1e-12)
    import jsonschema
    jsonschema.validate(ours, rcli.REPORT_SCHEMAS["plan"])


def test_profile_json_round_trip():
    from paper_2506_22175_b200.spec import HardwareProfile, SlowdownTable
    hw = HardwareProfile(1e14, 2e11, 3e10, SlowdownTable.from_factors(sigma_mem=0.9, mu_comp=0.7),
                         launch_overhead=1e-6, compute_saturation=64)
    assert cli.profile_from_json(cli.profile_to_json(hw)) == hw


@pytest.mark.parametrize("argv,code,kind", [
    (["memory", "--preset", "moe-bert-l", "--n", "2"], 2, "config"),          # no --batch
    (["memory", "--preset", "nope", "--batch", "8", "--n", "2"], 2, "usage"),  # bad choice
    (["memory", "--batch", "8", "--n", "x"], 2, "config"),
    (["plan", "--batch", "64", "--n", "2", "--hardware", "/nonexistent.json"], 2, "config"),
    (["memory", "--batch", "4", "--n", "8"], 1, "InvalidPartitioningError"),   # n > B
])
def test_errors_are_json(capsys, argv, code, kind):
    rc, _, err = _run(capsys, argv)
    assert rc == code
    body = json.loads(err.strip().splitlines()[-1])
    assert body["error"] == kind and body["message"]


def test_unknown_config_key(tmp_path, capsys):
    cf = tmp_path / "c.json"
    cf.write_text(json.dumps({"tokens": 64, "bogus": 1}))
    rc, _, err = _run(capsys, ["memory", "--config", str(cf), "--n", "2"])
    assert rc == 2 and json.loads(err)["path"] == "bogus"


@pytest.mark.gpu
def test_run_sweep_search_on_gpu(tmp_path, capsys):
    rcli = None
    try:
        rcli = _ref_cli()
    except pytest.skip.Exception:
        pass
    small = ["--model-dim", "256", "--hidden-dim", "512", "--num-experts", "8", "--top-k", "2"]
    trace = tmp_path / "t.jsonl"
    rc, out, err = _run(capsys, ["run", *small, "--batch", "4096", "--n", "4", "--strategy", "s4",
                                 "--out", str(trace)])
    assert rc == 0, err
    body = json.loads(out)
    assert body["makespan_us"] > 0 and body["reuse"] is True and set(body["busy_us"]) == {"compute", "collective", "copy"}
    assert len(trace.read_text().splitlines()) == body["ops"]
    rc, out, err = _run(capsys, ["sweep", *small, "--batches", "2048,4096", "--ns", "1,2", "--strategies", "none,s4"])
    assert rc == 0, err
    rows = list(csv.DictReader(io.StringIO(out)))
    assert len(rows) == 8 and all(int(r["makespan_us"]) > 0 for r in rows)
    rc, out, err = _run(capsys, ["search", *small, "--iterations", "6", "--b-min", "1024", "--b-max", "4096",
                                 "--step", "1024", "--n", "1"])
    assert rc == 0, err
    summary = json.loads(out)
    assert summary["iterations"] == 6 and summary["total_searches"] >= 1
    if rcli is not None:
        import jsonschema
        jsonschema.validate(body, rcli.REPORT_SCHEMAS["simulate"])
        jsonschema.validate(summary, rcli.REPORT_SCHEMAS["search_summary"])


def test_layer_rejects_shapes_without_a_kernel_path():
    """Unsupported shapes fail at construction with a clear message, before any device work."""
    import torch

    from paper_2506_22175_b200.layer import MoELayer
    with pytest.raises(ValueError, match="multiples of 32"):
        MoELayer(100, 256, 8, dtype=torch.bfloat16, device="cpu")
    with pytest.raises(ValueError, match="bfloat16 or float32"):
        MoELayer(128, 256, 8, dtype=torch.float16, device="cpu")
