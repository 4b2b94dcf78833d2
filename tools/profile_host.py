"""Host-side cost of issuing one layer step vs its GPU time (GPU box)."""
import sys, time, cProfile, pstats
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2506_22175_b200.layer import MoELayer

dev = torch.device("cuda", 0)
layer = MoELayer(1024, 4096, 64, top_k=2, pipeline=int(sys.argv[1]) if len(sys.argv) > 1 else 1,
                 dtype=torch.bfloat16, device=dev)
x = torch.randn(16384, 1024, device=dev).bfloat16().requires_grad_(True)
dy = torch.randn(16384, 1024, device=dev).bfloat16()
def step():
    y = layer(x); y.backward(dy); x.grad = None
    for p in layer.parameters(): p.grad = None
for _ in range(3): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3*(t1-t0)/10:.3f} ms/step, wall incl. drain {1e3*(t2-t0)/10:.3f} ms/step")
pr = cProfile.Profile(); pr.enable()
for _ in range(5): step()
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
