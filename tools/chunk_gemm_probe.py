"""Device time of one chunk's forward expert GEMMs (fc1 + ReLU-mask, fc2) at the
N=8 per-GPU shape (8 local experts, M=1024, H=4096) as the chunk shrinks: rows
per expert 4096 / n for n = 1, 2, 4, 8.  Back-to-back launches captured in a
CUDA graph (no host cost, no cross-stream events), so the difference to n x the
n=1 time is the GEMM's own per-launch and wave-quantisation cost."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
E, M, H, R = 8, 1024, 4096, 4096
bf = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.1).bfloat16()
x, w1, w2 = bf(E, R, M), bf(E, H, M), bf(E, M, H)
tm, do = bf(E, R, H), bf(E, R, M)
mask = torch.empty(E, R, H // 32, device=dev, dtype=torch.int32)


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    gr.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for n in (1, 2, 4, 8):
    r = R // n

    def chunks(r=r, n=n):
        for i in range(n):
            sl = slice(i * r, (i + 1) * r)
            ops.gemm(x[:, sl], w1, tm[:, sl], epilogue=_lib.EPI_RELU_MASK, aux=mask[:, sl])
            ops.gemm(tm[:, sl], w2, do[:, sl])

    def fc1(r=r, n=n):
        for i in range(n):
            sl = slice(i * r, (i + 1) * r)
            ops.gemm(x[:, sl], w1, tm[:, sl], epilogue=_lib.EPI_RELU_MASK, aux=mask[:, sl])

    def fc2(r=r, n=n):
        for i in range(n):
            sl = slice(i * r, (i + 1) * r)
            ops.gemm(tm[:, sl], w2, do[:, sl])

    side = torch.cuda.Stream()

    def two_streams(r=r, n=n):  # chunk i+1's fc1 on a second stream beside chunk i's fc2
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        evs = []
        for i in range(n):
            sl = slice(i * r, (i + 1) * r)
            s_ = side if i % 2 else cur
            with torch.cuda.stream(s_):
                ops.gemm(x[:, sl], w1, tm[:, sl], epilogue=_lib.EPI_RELU_MASK, aux=mask[:, sl])
                ops.gemm(tm[:, sl], w2, do[:, sl])
        cur.wait_stream(side)

    print(f"n={n} rows/expert {r:5d}: fc1+fc2 all chunks {graph_time(chunks):7.1f} us   "
          f"fc1 {graph_time(fc1):7.1f}   fc2 {graph_time(fc2):7.1f}   chunks alternating over two streams "
          f"{graph_time(two_streams):7.1f}", flush=True)
