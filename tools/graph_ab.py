"""Interleaved eager vs whole-step CUDA-graph timing (cfg2 layer, N=1), medians over rounds."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402
from paper_2506_22175_b200.spec import NO_REUSE, ReuseStrategy  # noqa: E402

dev = torch.device("cuda", 0)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
strat = ReuseStrategy.by_name(sys.argv[3]) if len(sys.argv) > 3 else NO_REUSE
E = int(sys.argv[4]) if len(sys.argv) > 4 else 64  # 8: the N=8 per-GPU expert count
M = int(sys.argv[5]) if len(sys.argv) > 5 else 1024  # configs[2]: 2048 8192 1
H = int(sys.argv[6]) if len(sys.argv) > 6 else 4096
K = int(sys.argv[7]) if len(sys.argv) > 7 else 2
layer = MoELayer(M, H, E, top_k=K, pipeline=n, dtype=torch.bfloat16, device=dev)
x = torch.randn(T, M, device=dev).bfloat16()
dy = torch.randn(T, M, device=dev).bfloat16()
sg = layer.step_graph(T, n, strat)
sg.x.copy_(x)  # the graph's static inputs (captured on zeros: all-tie routing would keep 2 experts busy)
sg.dy.copy_(dy)


def timed(fn, reps=30):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


eager_fn = lambda: layer.run_step(x, dy, n, strat)
for _ in range(5):
    eager_fn(); sg.replay()
res = {"eager": [], "graph": []}
for _ in range(7):
    res["eager"].append(timed(eager_fn))
    res["graph"].append(timed(sg.replay))
print(f"T={T} E={E} n={n} {strat.name}: eager median {statistics.median(res['eager']):.3f} ms "
      f"{[round(v, 3) for v in res['eager']]} | graph median {statistics.median(res['graph']):.3f} ms "
      f"{[round(v, 3) for v in res['graph']]}")
