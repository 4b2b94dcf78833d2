"""Effective SM clock at microsecond scale while fwd+bwd steps run back to back (BASELINE configs[1]
shape, N = 1): one co-resident warp records (globaltimer, clock64) every few microseconds
(mpm_clock_trace), and the layer's phase marks give the step boundaries.  Answers whether the
expert GEMMs slow down in a real step (vs ncu's serialised replays) because the SM clock drops
under the step's power draw.

  python tools/clock_trace.py [--steps 10] [--interval-us 5] [--cool 2]
"""
import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import _lib  # noqa: E402
from paper_2506_22175_b200.layer import MoELayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--interval-us", type=float, default=5.0)
    ap.add_argument("--cool", type=float, default=2.0)
    ap.add_argument("--E", type=int, default=64)
    ap.add_argument("--bucket-us", type=float, default=100.0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    T, M, H, k = 16384, 1024, 4096, 2
    layer = MoELayer(M, H, a.E, top_k=k, capacity_factor=1.0, pipeline=1, dtype=torch.bfloat16, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(T, M, device=dev, generator=g).bfloat16().requires_grad_(True)
    dy = torch.randn(T, M, device=dev, generator=g).bfloat16()

    def step():
        layer(x).backward(dy)
        x.grad = None
        for p in layer.parameters():
            p.grad = None

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    n = int(a.steps * 1600 / a.interval_us) + 400
    buf = torch.zeros(2 * n, dtype=torch.int64, device=dev)
    side = torch.cuda.Stream(device=dev)
    time.sleep(a.cool)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    _lib.call("mpm_clock_trace", ctypes.c_void_p(buf.data_ptr()), n, int(a.interval_us * 1000),
              ctypes.c_void_p(side.cuda_stream))
    time.sleep(0.001)
    ev[0].record()
    for i in range(a.steps):
        step()
        ev[i + 1].record()
    torch.cuda.synchronize()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.steps)]
    tr = buf.view(n, 2).cpu().tolist()
    t0 = tr[0][0]
    # MHz per bucket
    rows, j = [], 0
    bucket_ns = a.bucket_us * 1000
    while j < n - 1:
        jj = j
        while jj < n - 1 and tr[jj][0] - tr[j][0] < bucket_ns:
            jj += 1
        dt, dc = tr[jj][0] - tr[j][0], tr[jj][1] - tr[j][1]
        if dt <= 0:
            break
        rows.append((round((tr[j][0] - t0) / 1000, 1), round(dc / dt * 1000, 1)))
        j = jj
    mhz = [r[1] for r in rows]
    print(json.dumps({"step_ms": [round(v, 4) for v in step_ms], "trace_span_ms": round((tr[-1][0] - t0) / 1e6, 3),
                      "mhz_min": min(mhz), "mhz_max": max(mhz), "mhz_mean": round(sum(mhz) / len(mhz), 1)}))
    for t_us, f in rows:
        print(f"{t_us:9.1f} us  {f:7.1f} MHz")


if __name__ == "__main__":
    main()
