"""Measured schedule-DAG timeline of one fwd+bwd step (per-op CUDA events on each op's stream):
op, stream / lane, start and end in microseconds from the step origin, plus the phase marks.

  python tools/timeline.py [--E 8 --T 16384 --n 4 --strategy s4] [--trace out.json]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402
from paper_2506_22175_b200.trace import to_trace_event  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=1024)
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--strategy", default="s4")
    ap.add_argument("--trace", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    layer = MoELayer(a.M, a.H, a.E, top_k=a.k, pipeline=a.n, dtype=torch.bfloat16, device=dev)
    layer.record_times = True
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(a.T, a.M, device=dev, generator=g).bfloat16().requires_grad_(True)
    dy = torch.randn(a.T, a.M, device=dev, generator=g).bfloat16()
    strat = None if a.strategy == "none" else a.strategy
    for _ in range(4):
        layer(x, n=a.n, strategy=strat).backward(dy)
    torch.cuda.synchronize()
    ar = layer.last_arena
    fw, bw = ar.traces()
    for name, tr in (("forward", fw), ("backward", bw)):
        print(f"== {name}: makespan {tr.makespan * 1e6:.1f} us")
        for e in sorted(tr.events, key=lambda e: e.start):
            lane = tr.lanes.get(e.op_id, 0) if hasattr(tr, "lanes") else 0
            print(f"  {e.op_id:8s} {e.stream:10s} lane{lane} {e.start * 1e6:8.1f} {e.end * 1e6:8.1f} "
                  f"({(e.end - e.start) * 1e6:7.1f})")
    print("phases", json.dumps(ar.phase_ms()), "wgrad_ms", ar.wgrad_seconds() * 1e3)
    if a.trace:
        Path(a.trace).write_text(json.dumps({"forward": to_trace_event(fw), "backward": to_trace_event(bw)}))


if __name__ == "__main__":
    main()
