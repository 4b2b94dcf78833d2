"""BASELINE configs[3] step time (M=4096, H=16384, E=64 top-2, 393K tokens, N=1) under A/B switches, with
the SM clock and throttle reasons sampled during the timed steps.  Used to check the round-2 memory sweep
(`tools/sweep.py memory`) against round 1's.

  MPM_COMPUTE_LANES=1 / MPM_COMPACT=0 python tools/cfg4_probe.py [--n 8] [--strategy none] [--steps 2]
      [--tokens T --M --H --E --k]   (other shapes, e.g. configs[2]: --M 2048 --H 8192 --E 32 --k 1)
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2506_22175_b200.layer import MoELayer  # noqa: E402
from paper_2506_22175_b200.spec import NO_REUSE, ReuseStrategy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--strategy", default="none")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--tokens", type=int, default=393216)
ap.add_argument("--M", type=int, default=4096)
ap.add_argument("--H", type=int, default=16384)
ap.add_argument("--E", type=int, default=64)
ap.add_argument("--k", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
M, H, E, k, T = a.M, a.H, a.E, a.k, a.tokens
layer = MoELayer(M, H, E, top_k=k, capacity_factor=1.0, pipeline=a.n, dtype=torch.bfloat16, device=dev)
strat = NO_REUSE if a.strategy == "none" else ReuseStrategy.by_name(a.strategy)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, M, device=dev, generator=g).bfloat16()
dy = torch.randn(T, M, device=dev, generator=g).bfloat16()
layer.run_step(x, dy, a.n, strat)
torch.cuda.synchronize()
s = ClockSampler(dev.index)
s.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.monotonic()
e0.record()
for _ in range(a.steps):
    layer.run_step(x, dy, a.n, strat)
e1.record()
torch.cuda.synchronize()
clk = s.stop((w0, time.monotonic()))
ms = e0.elapsed_time(e1) / a.steps
flops = 12 * k * T * M * H
print(json.dumps({"M": M, "H": H, "E": E, "k": k, "n": a.n, "strategy": a.strategy, "tokens": T, "ms_per_step": round(ms, 1),
                  "expert_tflops": round(flops / ms / 1e9, 1), "lanes": os.environ.get("MPM_COMPUTE_LANES"),
                  "compact": os.environ.get("MPM_COMPACT"), "clocks": clk}), flush=True)
