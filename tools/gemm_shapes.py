"""Characterise the tcgen05 GEMM across shapes/layouts (CUDA events, 20 reps):
which of K-length, output size, grouping (batches) and operand majorness
costs throughput.  cuBLAS (torch.bmm / matmul) on the same shapes beside it."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)


def bf(*s):
    return (torch.randn(*s, device=dev, generator=g) * 0.1).bfloat16()


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


CASES = [  # name, batches, rows, N, K, a_mn, b_mn
    ("fc1_fwd 64x512x4096x1024", 64, 512, 4096, 1024, False, False),
    ("fc2_fwd 64x512x1024x4096", 64, 512, 1024, 4096, False, False),
    ("wgrad_mn 64x4096x1024x512", 64, 4096, 1024, 512, True, True),
    ("wgrad_kmaj 64x4096x1024x512", 64, 4096, 1024, 512, False, False),
    ("wgrad_K1024 64x4096x1024x1024", 64, 4096, 1024, 1024, True, True),
    ("wgrad_K4096 8x4096x1024x4096", 8, 4096, 1024, 4096, True, True),
    ("single 1x32768x4096x1024", 1, 32768, 4096, 1024, False, False),
    ("single 1x8192x8192x8192", 1, 8192, 8192, 8192, False, False),
    ("fc1 N8 8x4096x4096x1024", 8, 4096, 4096, 1024, False, False),
]
for name, B, R, N, K, amn, bmn in CASES:
    a = bf(B, K, R) if amn else bf(B, R, K)
    b = bf(B, K, N) if bmn else bf(B, N, K)
    c = torch.empty(B, R, N, device=dev, dtype=torch.bfloat16)
    t = timeit(lambda: ops.gemm(a, b, c, a_mn_major=amn, b_mn_major=bmn))
    A = a.transpose(1, 2) if amn else a
    Bt = b if bmn else b.transpose(1, 2)
    tc = timeit(lambda: torch.bmm(A, Bt, out=c))
    f = 2.0 * B * R * N * K
    print(f"{name:34s} ours {t * 1e6:8.1f} us {f / t / 1e12:7.1f} TF/s   cublas {tc * 1e6:8.1f} us {f / tc / 1e12:7.1f} TF/s")
