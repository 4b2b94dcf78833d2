"""Does the exchange copy kernel run *beside* a persistent expert GEMM?

Launches a long tcgen05 GEMM (cfg2 fc2 shape, every SM busy) on stream A and,
while it runs, one N=8-shaped p2p copy exchange (SM copy kernel) on stream B.
If the copy kernel fits next to the GEMM CTAs it finishes long before the
GEMM; if it needed the GEMM's SMs it would end after it.  Also reports how
much the GEMM slows down with the copy running beside it, and the same for
a copy-engine exchange (MPM_P2P_COPY=serial)."""
import ctypes
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
E, R, M, H = 64, 512, 1024, 4096
g = torch.Generator(device=dev).manual_seed(0)
tm = (torch.randn(E, R, H, device=dev, generator=g) * 0.1).bfloat16()
w2 = (torch.randn(E, M, H, device=dev, generator=g) * 0.1).bfloat16()
out = torch.empty(E, R, M, device=dev, dtype=torch.bfloat16)

N, E_LOC, C_I = 8, 8, 128
rb = M * 2
bufs = [torch.zeros(E_LOC * C_I * 8 * rb, device=dev, dtype=torch.uint8) for _ in range(N)]
dst = torch.zeros(E_LOC * N * C_I * rb, device=dev, dtype=torch.uint8)
flags = torch.zeros(64, device=dev, dtype=torch.int32)
counter = torch.zeros(1, device=dev, dtype=torch.int32)
plan = _lib.P2PPlan()
plan.n_copy = N
for p in range(N):
    c = plan.copy[p]
    c.dst, c.src = dst.data_ptr() + p * C_I * rb, bufs[p].data_ptr()
    c.dpitch, c.spitch, c.width, c.height = N * C_I * rb, 8 * C_I * rb, C_I * rb, E_LOC
plan.n_signal = N - 1
for j in range(N - 1):
    plan.signal[j] = flags.data_ptr() + 4 * j
plan.counter = counter.data_ptr()
epoch = ctypes.c_uint32(0)
lib = _lib.load()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def gemm():
    ops.gemm(tm, w2, out, stream=sa)


def exchange():
    epoch.value += 1
    assert lib.mpm_p2p_run(ctypes.byref(plan), epoch, ctypes.c_void_p(sb.cuda_stream)) == 0, lib.mpm_last_error()


def timed(fn_list):
    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in fn_list}
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(sa)
    sb.wait_event(t0)
    for name, (fn, st) in fn_list.items():
        ev[name][0].record(st)
        fn()
        ev[name][1].record(st)
    torch.cuda.synchronize()
    return {k: (t0.elapsed_time(a) * 1e3, t0.elapsed_time(b) * 1e3) for k, (a, b) in ev.items()}


for _ in range(3):
    gemm()
    exchange()
torch.cuda.synchronize()
alone_g = timed({"gemm": (gemm, sa)})["gemm"]
alone_x = timed({"copy": (exchange, sb)})["copy"]
both = timed({"gemm": (gemm, sa), "copy": (exchange, sb)})
print(json.dumps({"copy_mode": os.environ.get("MPM_P2P_COPY", "sm"),
                  "gemm_alone_us": alone_g[1] - alone_g[0], "copy_alone_us": alone_x[1] - alone_x[0],
                  "together": {k: {"start_us": round(a, 1), "end_us": round(b, 1)} for k, (a, b) in both.items()},
                  "copy_finished_before_gemm": both["copy"][1] < both["gemm"][1],
                  "gemm_slowdown": (both["gemm"][1] - both["gemm"][0]) / (alone_g[1] - alone_g[0])}))
