"""Where does the CUDA-graph gain come from?  Eager vs graph time of the forward and the backward of
one cfg2 step (N=1) captured separately (static inputs/outputs; measurement only)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer, _Arena  # noqa: E402
from paper_2506_22175_b200.spec import NO_REUSE  # noqa: E402

dev = torch.device("cuda", 0)
T = 16384
layer = MoELayer(1024, 4096, 64, top_k=2, pipeline=1, dtype=torch.bfloat16, device=dev)
x = torch.randn(T, 1024, device=dev).bfloat16()
dy = torch.randn(T, 1024, device=dev).bfloat16()
arena = _Arena(layer, T, 1, NO_REUSE, False, torch.bfloat16, False)


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


side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    arena.forward(x)
    arena.backward(x, dy)
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.graph(gf):
    arena.forward(x)
with torch.cuda.graph(gb):
    arena.backward(x, dy)
fe = timed(lambda: arena.forward(x))
fg = timed(gf.replay)
be = timed(lambda: arena.backward(x, dy))
bg = timed(gb.replay)
print(f"forward eager {fe:.3f} graph {fg:.3f} ms | backward eager {be:.3f} graph {bg:.3f} ms")

# whole step in one graph vs the two graphs back to back, and bitwise equality at this size
sg = layer.step_graph(T, 1, NO_REUSE)
both = timed(lambda: (gf.replay(), gb.replay()))
whole = timed(sg.replay)
eager = timed(lambda: layer.run_step(x, dy, 1, NO_REUSE))
y_e, g_e = layer.run_step(x, dy, 1, NO_REUSE)
y_g, g_g = sg.replay(x, dy)
torch.cuda.synchronize()
same = torch.equal(y_e, y_g) and all(torch.equal(a, b) for a, b in zip(g_e, g_g))
print(f"eager step {eager:.3f} | fwd graph + bwd graph {both:.3f} | whole-step graph {whole:.3f} ms | bitwise equal: {same}")
