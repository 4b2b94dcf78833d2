"""Times the forward gate front end at cfg2/N=1 (T=16K, M=1024, E=64): the fused
gate_route call and its gate GEMM alone ([T, M] x [3E, M]^T -> [T, 3E] f32) at
several tile shapes (N split into 64/128-wide slices to emulate narrower tiles).
Warm-L2 device timing (CUDA graph of back-to-back calls, CUDA events), as inside a step.  `MPM_GEMM_PAIR=0` selects
single-CTA tiles for the full-width case."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import _lib, ops  # noqa: E402

T, M, E, k = 16384, 1024, 64, 2
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, M, device=dev, generator=g).bfloat16()
wg = torch.randn(E, M, device=dev, generator=g) / 32
w3 = torch.randn(3 * E, M, device=dev, generator=g).bfloat16()
part = torch.empty(T, 3 * E, device=dev)


def timeit(fn, reps=50):
    """Device time per call: `reps` calls captured in one CUDA graph (no host issue cost)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(reps):
            fn()
    graph.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    graph.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


out = ops.gate_route(x, wg, k)
gws = ops.gate_workspace(T, M, E, dev)
print(f"gate_route           {timeit(lambda: ops.gate_route(x, wg, k, out=out, gate_ws=gws)):7.1f} us")
print(f"gemm n=192           {timeit(lambda: ops.gemm(x[None], w3[None], part[None], epilogue=_lib.EPI_STORE_F32)):7.1f} us")
for w in (64, 128):
    def sl(w=w):
        for j in range(0, 3 * E, w):
            ops.gemm(x[None], w3[None, j:j + w], part[None, :, j:j + w], epilogue=_lib.EPI_STORE_F32)
    print(f"gemm 3E/{w} slices    {timeit(sl):7.1f} us")
print(f"x read alone (copy)  {timeit(lambda: x.clone()):7.1f} us")
