"""Interleaved A/B of one vs two compute lanes for the chunked pipeline at the N=8
per-GPU shape (8 local experts, 16K tokens, top-2; no reuse): median fwd+bwd step
over rounds, same process, arenas rebuilt per setting."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402

dev = torch.device("cuda", 0)
E = int(sys.argv[1]) if len(sys.argv) > 1 else 8
layer = MoELayer(1024, 4096, E, top_k=2, pipeline=1, dtype=torch.bfloat16, device=dev)
x = torch.randn(16384, 1024, device=dev).bfloat16().requires_grad_(True)
dy = torch.randn(16384, 1024, device=dev).bfloat16()


def step(n):
    y = layer(x, n=n)
    y.backward(dy)
    x.grad = None
    for p in layer.parameters():
        p.grad = None


def timed(n, reps=15):
    for _ in range(3):
        step(n)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        step(n)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for n in (2, 4, 8):
    res = {1: [], 2: []}
    for _ in range(5):
        for lanes in (1, 2):
            layer.compute_lanes = lanes
            layer.release_arenas()
            res[lanes].append(timed(n))
    print(f"E={E} n={n}: one lane {statistics.median(res[1]):.3f} ms {[round(v, 3) for v in res[1]]} | "
          f"two lanes {statistics.median(res[2]):.3f} ms {[round(v, 3) for v in res[2]]}", flush=True)
