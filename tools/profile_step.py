"""Steady-state cfg2 steps (N=1) bracketed for ncu: warm-up outside, then
cudaProfilerStart / two autograd fwd+bwd steps / cudaProfilerStop.  Use with
`ncu --profile-from-start off ...` so the capture holds exactly the steady-state
launches (no planning trials, no arena construction)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402

dev = torch.device("cuda", 0)
T = 16384
E = int(sys.argv[2]) if len(sys.argv) > 2 else 64  # 8 = the expert count one rank owns at N=8
layer = MoELayer(1024, 4096, E, top_k=2, capacity_factor=1.0, pipeline=1, dtype=torch.bfloat16, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, 1024, device=dev, generator=g).bfloat16().requires_grad_(True)
dy = torch.randn(T, 1024, device=dev, generator=g).bfloat16()


def step():
    y = layer(x)
    y.backward(dy)
    x.grad = None
    for p in layer.parameters():
        p.grad = None


for _ in range(5):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
