"""One small forward + backward of the layer (and a reuse-strategy step) for compute-sanitizer runs:
  compute-sanitizer --tool memcheck python tools/sanitize_step.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402
from paper_2506_22175_b200.spec import NO_REUSE, ReuseStrategy  # noqa: E402

dev = torch.device("cuda", 0)
layer = MoELayer(256, 512, 8, top_k=2, capacity_factor=1.25, pipeline=2, dtype=torch.bfloat16, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(300, 256, device=dev, generator=g).bfloat16()
dy = torch.randn(300, 256, device=dev, generator=g).bfloat16()
for n, strat in ((1, NO_REUSE), (2, ReuseStrategy.by_name("s4")), (3, ReuseStrategy.by_name("s1"))):
    y, grads = layer.run_step(x, dy, n, strat)
torch.cuda.synchronize()
# padded tensor-core gate (E % 32 != 0) forward and backward (T % 64 == 0), E % 4 != 0
for E, T in ((8, 512), (6, 256), (64, 1024)):
    lay = MoELayer(256, 512, E, top_k=2, pipeline=1, dtype=torch.bfloat16, device=dev)
    xe = torch.randn(T, 256, device=dev, generator=g).bfloat16().requires_grad_(True)
    lay(xe).float().sum().backward()
torch.cuda.synchronize()
layer32 = MoELayer(256, 512, 4, top_k=1, pipeline=2, dtype=torch.float32, device=dev)
x32 = torch.randn(256, 256, device=dev).requires_grad_(True)
layer32(x32).sum().backward()
torch.cuda.synchronize()
print("sanitize step ok")
