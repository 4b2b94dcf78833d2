"""Generates tests/golden/data_plane.json: frozen data-plane vectors of the CPU oracle.

The reference has no MoE numerics (data-plane parity is unpinned
by the reference), so the oracle's own outputs on seeded inputs are frozen here
to pin its semantics across versions: BASELINE.json configs[0] (4 experts top-1,
M=256, H=1024, 2048 tokens, n=2, fp32) and a top-2 two-rank case with capacity
drops.  Stored: the full routing (indices, slots, kept counts — exact) and
fingerprints of every float output (sum, |sum|, L2 norm, 16 fixed entries —
compared with a tight tolerance).  Inputs are regenerated from the seeds by
`make_inputs` (numpy PCG64), so the fixture stays small.

    python tests/golden/gen_data_plane.py      # rewrites the fixture
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import moe_oracle as O  # noqa: E402

CASES = {
    "cfg1_fp32": dict(N=1, T=2048, M=256, H=1024, E=4, k=1, cf=1.0, n=2, seed=1),
    "top2_two_rank_drops": dict(N=2, T=300, M=64, H=128, E=8, k=2, cf=0.75, n=3, seed=2),
}


def make_inputs(c: dict):
    rng = np.random.default_rng(c["seed"])
    N, T, M, H, E = c["N"], c["T"], c["M"], c["H"], c["E"]
    xs = [rng.standard_normal((T, M)).astype(np.float32) for _ in range(N)]
    dys = [rng.standard_normal((T, M)).astype(np.float32) for _ in range(N)]
    wg = (rng.standard_normal((E, M)) / np.sqrt(M)).astype(np.float32)
    w1s = [(rng.standard_normal((E // N, H, M)) * 0.05).astype(np.float32) for _ in range(N)]
    w2s = [(rng.standard_normal((E // N, M, H)) * 0.05).astype(np.float32) for _ in range(N)]
    return xs, dys, wg, w1s, w2s


def run(c: dict):
    xs, dys, wg, w1s, w2s = make_inputs(c)
    return O.moe_layer(xs, wg, w1s, w2s, k=c["k"], capacity_factor=c["cf"], n_chunks=c["n"], dys=dys)


def fingerprint(a) -> dict:
    a = np.asarray(a, dtype=np.float64).ravel()
    pick = np.linspace(0, a.size - 1, 16).astype(np.int64)
    return {"sum": float(a.sum()), "abs_sum": float(np.abs(a).sum()), "l2": float(np.sqrt((a * a).sum())),
            "samples": [float(v) for v in a[pick]]}


def summarize(c: dict) -> dict:
    res = run(c)
    out = {"case": c, "routing": [], "y": [], "dx": [], "dw1": [], "dw2": [], "dwg": fingerprint(res.dwg)}
    for r in range(c["N"]):
        rt = res.routing[r]
        out["routing"].append({"idx": rt.idx.tolist(), "slot": rt.slot.tolist(), "kept": rt.kept.tolist()})
        for key in ("y", "dx", "dw1", "dw2"):
            out[key].append(fingerprint(getattr(res, key)[r]))
    return out


if __name__ == "__main__":
    data = {name: summarize(c) for name, c in CASES.items()}
    (Path(__file__).parent / "data_plane.json").write_text(json.dumps(data))
    print("wrote", Path(__file__).parent / "data_plane.json")
