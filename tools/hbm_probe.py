"""Times the HBM-bound routing kernels of one cfg2 step at N=1 (T=16K, M=1024,
E=64, top-2, cf 1.0) in isolation: CUDA-event time per launch and algorithmic
GB/s (bytes a perfect kernel must move), against the measured
HBM copy peak.  MPM_LIB=... selects another libmpm build (A/B)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import ops  # noqa: E402

T, M, E, k = 16384, 1024, 64, 2
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, M, device=dev, generator=g).bfloat16()
wg = torch.randn(E, M, device=dev, generator=g) / 32
C = ops.capacity(T, k, E, 1.0)
r = ops.compute_routing(x, wg, k, C, True)
t_i = torch.empty(E * C, M, device=dev, dtype=torch.bfloat16)
t_o = torch.randn(E * C, M, device=dev, generator=g).bfloat16()
g_o = torch.empty_like(t_o)
g_i = torch.randn(E * C, M, device=dev, generator=g).bfloat16()
dy = torch.randn(T, M, device=dev, generator=g).bfloat16()
dprob = torch.empty(T, k, device=dev)
dl = torch.randn(T, E, device=dev, generator=g) * 1e-3
ws = ops.gate_workspace(T, M, E, dev)
dx = torch.empty(T, M, device=dev, dtype=torch.bfloat16)
y = torch.empty(T, M, device=dev, dtype=torch.bfloat16)
logits = torch.empty(T, E, device=dev)
dlg = torch.zeros(T, E, device=dev)
dwg = torch.empty(E, M, device=dev)
row = M * 2
rws = torch.empty(int(ops._lib.load().mpm_route_workspace_bytes(T, E, k)), device=dev, dtype=torch.uint8)
ridx = torch.empty(T, k, device=dev, dtype=torch.int32)
rw = torch.empty(T, k, device=dev)
rslot = torch.empty(T, k, device=dev, dtype=torch.int32)
rkept = torch.empty(E, device=dev, dtype=torch.int32)
cases = {
    "route": (lambda: ops.route(r.logits, k, True, out=(ridx, rw, rws)), T * E * 4 + T * k * 8),
    "assign_slots": (lambda: ops.assign_slots(ridx, E, C, rws, out=(rslot, rkept)), T * k * 8),
    "gate_fwd": (lambda: ops.gate_fwd(x, wg, out=logits, ws=ws), T * row + T * E * 4),
    "gate_fwd+route": (lambda: (ops.gate_fwd(x, wg, out=logits, ws=ws), ops.route(logits, k, True, out=(ridx, rw, rws))),
                       T * row + T * E * 4 + T * k * 8),
    "gate_route": (lambda: ops.gate_route(x, wg, k, True, out=(logits, ridx, rw, rws), gate_ws=ws),
                   T * row + T * E * 4 + T * k * 8),
    "permute": (lambda: ops.permute(x, r, 1, t_i), T * row + E * C * row),
    "combine": (lambda: ops.combine(t_o, r, 1, T, out=y), T * k * row + T * row),
    "combine_bwd": (lambda: ops.combine_bwd(dy, t_o, r, 1, g_o, out=dprob), T * row + T * k * row + E * C * row),
    "gather_bwd": (lambda: ops.gather_bwd(g_i, r, dl, wg, 1, T), 2 * T * row + T * k * row),
    # the layer's backward kernels at N=1: combine backward fused with the gate softmax backward
    # (dy + k T_O rows in, k g_o rows + dlogits + split operands out; the unused slots' zero rows), the
    # dWg GEMM + split reduce, and the gather with the sparse gate term (k g_i rows in, dx out)
    "combine_bwd_gate": (lambda: ops.combine_bwd_gate(dy, t_o, r, 1, g_o, dlg, ws, True),
                         T * row + 2 * T * k * row + T * E * 4),
    "gate_bwd_gemms": (lambda: ops.gate_backward_gemms(x, wg, dlg, k, True, dwg, dx, ws), T * row + E * M * 4),
    "gate_gather": (lambda: ops.gate_gather(r, g_i, wg, 1, dlg, True, dx, ws), T * k * row + T * row),
}
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6538.3) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6538.3
flush = torch.empty(256 * 1024 * 1024, device=dev, dtype=torch.uint8)
for name, (fn, nbytes) in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()  # cold L2 between launches (inputs > 126 MB L2 anyway for most)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b) * 1e-3
    t = tot / reps
    print(f"{name:12s} {t * 1e6:8.1f} us  {nbytes / t / 1e9:8.0f} GB/s  {nbytes / t / 1e9 / peak:5.2f} of HBM peak")
