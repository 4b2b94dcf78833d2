"""Runs the six expert GEMMs of one cfg2 step at N=1 (64 experts x 512 rows, M=1024,
H=4096) once each, for ncu captures and per-GEMM CUDA-event timing."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_22175_b200 import _lib, ops

E, R, M, H = 64, 512, 1024, 4096
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
bf = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.1).bfloat16()
x, w1, w2 = bf(E, R, M), bf(E, H, M), bf(E, M, H)
tm, do, dm, di = bf(E, R, H), bf(E, R, M), bf(E, R, H), bf(E, R, M)
dw1, dw2 = torch.empty_like(w1), torch.empty_like(w2)
mask = torch.empty(E, R, H // 32, device=dev, dtype=torch.int32)
acc = torch.zeros(E, M, H, device=dev)
cases = {
    "fc1_fwd": lambda: ops.gemm(x, w1, tm, epilogue=_lib.EPI_RELU_MASK, aux=mask),
    "fc1_fwd_plain": lambda: ops.gemm(x, w1, tm),  # the same GEMM without the ReLU / mask epilogue
    "fc2_fwd": lambda: ops.gemm(tm, w2, do),
    "fc2_dgrad_plain": lambda: ops.gemm(do, w2, dm, b_mn_major=True),
    "fc2_dgrad": lambda: ops.gemm(do, w2, dm, b_mn_major=True, epilogue=_lib.EPI_DMASK, aux=mask),
    "fc2_dgrad_aux": lambda: ops.gemm(do, w2, dm, b_mn_major=True, epilogue=_lib.EPI_DRELU, aux=tm),
    "fc1_dgrad": lambda: ops.gemm(dm, w1, di, b_mn_major=True),
    "fc2_wgrad": lambda: ops.gemm(do, tm, dw2, a_mn_major=True, b_mn_major=True),
    "fc1_wgrad": lambda: ops.gemm(dm, x, dw1, a_mn_major=True, b_mn_major=True),
    "wgrad_acc": lambda: ops.gemm(do, tm, acc, a_mn_major=True, b_mn_major=True, epilogue=_lib.EPI_ACCUM_F32),
    # cuBLAS on the same shapes (library ceiling for comparison, not a product path)
    "cublas_fc1_fwd": lambda: torch.bmm(x, w1.transpose(1, 2), out=tm),
    "cublas_fc2_fwd": lambda: torch.bmm(tm, w2.transpose(1, 2), out=do),
    "cublas_fc1_dgrad": lambda: torch.bmm(dm, w1, out=di),
    "cublas_fc2_wgrad": lambda: torch.bmm(do.transpose(1, 2), tm, out=dw2),
    "cublas_fc1_wgrad": lambda: torch.bmm(dm.transpose(1, 2), x, out=dw1),
}
flops = 2.0 * E * R * M * H
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for name, fn in cases.items():
    if only and name not in only:
        continue
    for _ in range(3 if reps > 1 else 1):  # reps == 1: exactly one launch per GEMM (ncu)
        fn()
    torch.cuda.synchronize()
    if reps <= 1:
        continue
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    print(f"{name:14s} {us:8.1f} us  {flops / us / 1e6:8.1f} TFLOP/s")
