"""StepGraph: one forward + backward captured as a CUDA graph replays bit-identically to the eager
step (every schedule-DAG op on three streams, the gate side stream, host offload copies) and costs
less time per step when the step is launch-bound."""

import pytest
import torch

from paper_2506_22175_b200.layer import MoELayer
from paper_2506_22175_b200.spec import NO_REUSE, ReuseStrategy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,strategy", [(1, None), (2, "s4"), (4, "s1"), (2, "s3"), (3, None)])  # (3, None): two compute lanes
def test_graph_replay_matches_eager(cuda, n, strategy):
    layer = MoELayer(256, 512, 8, top_k=2, pipeline=n, dtype=torch.bfloat16, device=cuda)
    strat = ReuseStrategy.by_name(strategy) if strategy else NO_REUSE
    g = torch.Generator(device=cuda).manual_seed(n)
    T = 1024
    xs = [torch.randn(T, 256, device=cuda, generator=g).bfloat16() for _ in range(2)]
    dys = [torch.randn(T, 256, device=cuda, generator=g).bfloat16() for _ in range(2)]
    sg = layer.step_graph(T, n, strat)
    for x, dy in zip(xs, dys):  # two different inputs through the same graph
        y_e, grads_e = layer.run_step(x, dy, n, strat)
        y_g, grads_g = sg.replay(x, dy)
        torch.cuda.synchronize()
        assert torch.equal(y_e, y_g)
        for a, b in zip(grads_e, grads_g):
            assert torch.equal(a, b)


def test_graph_is_faster_when_launch_bound(cuda):
    layer = MoELayer(256, 512, 8, top_k=2, pipeline=2, dtype=torch.bfloat16, device=cuda)
    T = 512
    x = torch.randn(T, 256, device=cuda).bfloat16()
    dy = torch.randn(T, 256, device=cuda).bfloat16()
    sg = layer.step_graph(T, 2, NO_REUSE)

    def timed(fn, reps=50):
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

    eager = timed(lambda: layer.run_step(x, dy, 2, NO_REUSE))
    graph = timed(lambda: sg.replay())
    assert graph < eager, (graph, eager)
