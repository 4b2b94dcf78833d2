"""Eager vs CUDA-graph step time (layer.StepGraph) across token counts at the cfg2 layer shape."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402
from paper_2506_22175_b200.spec import NO_REUSE  # noqa: E402

dev = torch.device("cuda", 0)
layer = MoELayer(1024, 4096, 64, top_k=2, pipeline=1, dtype=torch.bfloat16, device=dev)


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for T in (256, 1024, 4096, 16384):
    for n in (1, 4):
        x = torch.randn(T, 1024, device=dev).bfloat16()
        dy = torch.randn(T, 1024, device=dev).bfloat16()
        eager = timed(lambda: layer.run_step(x, dy, n, NO_REUSE))
        sg = layer.step_graph(T, n, NO_REUSE)
        graph = timed(lambda: sg.replay())
        print(f"T={T:6d} n={n}: eager {eager:7.3f} ms  graph {graph:7.3f} ms  ({eager / graph:4.2f}x)", flush=True)
        del sg
        layer.release_arenas()
