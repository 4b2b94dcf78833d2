"""Kernel-level timeline of steady-state fwd+bwd steps from CUPTI activity records (torch.profiler):
every kernel's stream, start and duration with concurrency intact (ncu serialises kernels; the
schedule-op events of tools/timeline.py only bracket ops).  Prints the last step's kernels in start
order with the idle gap before each on its stream and the busy union of all streams, so launch gaps,
ramp tails and side-stream overlap can be read directly.

  python tools/kernel_timeline.py [--E 64 --T 16384 --n 1 --strategy none] [--json out.json]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402


def short(name: str) -> str:
    name = name.replace("void ", "")
    for cut in ("(CUtensorMap", "(const", "(float", "(int", "(unsigned", "(__nv", "(sm100", "("):
        if cut in name:
            name = name[: name.index(cut)]
            break
    return name[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=1024)
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--E", type=int, default=64)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("--strategy", default="none")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--json", default=None)
    ap.add_argument("--serial-gather", action="store_true", help="gather after the weight gradients")
    ap.add_argument("--isolated", action="store_true",
                    help="synchronise + idle between profiled steps (default: back to back, as in bench.py)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    layer = MoELayer(a.M, a.H, a.E, top_k=a.k, pipeline=a.n, dtype=torch.bfloat16, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(a.T, a.M, device=dev, generator=g).bfloat16().requires_grad_(True)
    dy = torch.randn(a.T, a.M, device=dev, generator=g).bfloat16()
    strat = None if a.strategy == "none" else a.strategy
    layer._gather_side = not a.serial_gather

    def step():
        layer(x, n=a.n, strategy=strat).backward(dy)
        x.grad = None
        for p in layer.parameters():
            p.grad = None

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    time.sleep(1.0)  # cool down: the profiled steps run at boost clocks like the bench window
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            if a.isolated:
                torch.cuda.synchronize()
                time.sleep(0.005)
            step()
        torch.cuda.synchronize()
    kern = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0
            and "Memcpy" not in e.name and "Memset" not in e.name]
    kern.sort(key=lambda e: e.time_range.start)
    # every step launches the same kernels: the last step = the last len / steps kernels by start
    per_step = len(kern) // a.steps
    last = kern[len(kern) - per_step:]
    # per profiled step: span and the summed duration of the expert-GEMM-sized kernels (> 100 us),
    # to see clock drift across back-to-back steps (the step is power-limited under sustained load)
    first = len(kern) - per_step * a.steps
    drift = []
    for j in range(a.steps):
        ks = kern[first + j * per_step: first + (j + 1) * per_step]
        drift.append({"span_us": round(max(e.time_range.end for e in ks) - ks[0].time_range.start, 1),
                      "big_gemm_us": round(sum(e.time_range.elapsed_us() for e in ks
                                               if e.time_range.elapsed_us() > 100), 1)})
    print("per-step", json.dumps(drift))
    t0 = last[0].time_range.start
    rows, stream_end = [], {}
    busy, cur_s, cur_e = 0.0, None, None
    for e in last:
        s, d = e.time_range.start - t0, e.time_range.elapsed_us()
        st = getattr(e, "device_resource_id", None)
        gap = s - stream_end[st] if st in stream_end else 0.0
        stream_end[st] = s + d
        rows.append({"kernel": short(e.name), "stream": st, "start_us": round(s, 1), "dur_us": round(d, 1),
                     "gap_us": round(gap, 1)})
        if cur_s is None or s > cur_e:
            if cur_s is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, s + d
        else:
            cur_e = max(cur_e, s + d)
    busy += cur_e - cur_s
    span = max(r["start_us"] + r["dur_us"] for r in rows)
    for r in rows:
        print(f"{r['start_us']:8.1f} {r['dur_us']:7.1f} gap {r['gap_us']:6.1f}  s{r['stream']}  {r['kernel']}")
    summary = {"span_us": round(span, 1), "busy_union_us": round(busy, 1), "kernels": len(rows),
               "idle_us": round(span - busy, 1), "config": vars(a)}
    print(json.dumps(summary))
    if a.json:
        Path(a.json).write_text(json.dumps({"summary": summary, "kernels": rows}, indent=1))


if __name__ == "__main__":
    main()
