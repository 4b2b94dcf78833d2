"""Host and device cost of one mpm_p2p_run exchange (single GPU, single process).

Builds an N=8-shaped dispatch plan whose 'peer windows' are 8 local buffers:
7 flag waits (already satisfied), 8 copies of E_loc=8 rows x c_i*M*2 bytes,
7 flag stores, 7 arrival waits (satisfied by the stores).  Reports host
microseconds per call (the API cost the executor pays per exchange) and
device time per exchange with the copy fan-out on and off.  Local copies
run over HBM, not NVLink: the device numbers bound the copy-engine issue
overhead, not the link bandwidth.
"""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import _lib  # noqa: E402

N, E_LOC, C_I, M = 8, 8, 128, 1024
dev = torch.device("cuda", 0)
rb = M * 2
bufs = [torch.zeros(E_LOC * C_I * 8 * rb, device=dev, dtype=torch.uint8) for _ in range(N)]
dst = torch.zeros(E_LOC * N * C_I * rb, device=dev, dtype=torch.uint8)
flags = torch.zeros(64, device=dev, dtype=torch.int32)
plan = _lib.P2PPlan()
plan.n_wait = N - 1
for j in range(N - 1):
    plan.wait[j] = flags.data_ptr() + 4 * j
plan.n_copy = N
for p in range(N):
    c = plan.copy[p]
    c.dst, c.src = dst.data_ptr() + p * C_I * rb, bufs[p].data_ptr()
    c.dpitch, c.spitch, c.width, c.height = N * C_I * rb, 8 * C_I * rb, C_I * rb, E_LOC
plan.n_signal = N - 1
for j in range(N - 1):
    plan.signal[j] = flags.data_ptr() + 4 * (16 + j)
plan.n_arrive = N - 1
for j in range(N - 1):
    plan.arrive[j] = flags.data_ptr() + 4 * (16 + j)
counter = torch.zeros(1, device=dev, dtype=torch.int32)
plan.counter = counter.data_ptr()
epoch = ctypes.c_uint32(1)
flags[:8].fill_(1 << 30)  # "ready" waits always satisfied
stream = torch.cuda.Stream()  # the batched copy API refuses the legacy default stream
lib = _lib.load()


def run(k):
    for _ in range(k):
        rc = lib.mpm_p2p_run(ctypes.byref(plan), epoch, ctypes.c_void_p(stream.cuda_stream))
        assert rc == 0, lib.mpm_last_error()
        epoch.value += 1


run(20)
torch.cuda.synchronize()
t0 = time.perf_counter()
run(200)
t1 = time.perf_counter()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
run(200)
b.record(stream)
torch.cuda.synchronize()
moved = N * E_LOC * C_I * rb
print(f"copy={__import__('os').environ.get('MPM_P2P_COPY', 'sm')}: host {1e6 * (t1 - t0) / 200:.1f} us/call, "
      f"device {1e3 * a.elapsed_time(b) / 200:.1f} us/exchange, {moved / (a.elapsed_time(b) / 200 * 1e-3) / 1e9:.0f} GB/s "
      f"({moved / 1e6:.1f} MB per exchange)")
