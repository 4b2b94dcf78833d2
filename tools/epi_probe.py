"""Where the expert GEMMs' warp roles wait (needs a libmpm built with MPM_NVCC_FLAGS=-DMPM_EPI_PROBE).

Sums of SM-clock cycles over all CTAs, per launch:
  0 producer waiting for a free ring stage      1 MMA issuer waiting for a free accumulator (tempty)
  2 MMA issuer waiting for a loaded stage       3 epilogue warp waiting for an accumulator (tfull)
  4 epilogue tcgen05.ld (64 columns + wait)     5 epilogue waiting for its staging buffer (TMA store read)
  6 epilogue, accumulator ready -> released     7 epilogue tiles (warps x tiles)
  8 MMA issuer loop total                       9 entry -> after griddepcontrol.wait (MMA thread)
 10 routing epilogue (gate GEMM, per warp)     11 entry -> epilogue done (first epilogue warp)
 12-15 routing epilogue parts: TMEM loads, logits stores, top-k + softmax + idx/weights, block counts
Usage: python tools/epi_probe.py [case,...]   (cases of tools/gemm_probe.py)"""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2506_22175_b200 import _lib

lib = _lib.load()
fn = lib.mpm_debug_epi_probe
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()

cases = sys.argv[1].split(",") if len(sys.argv) > 1 else ["fc1_fwd", "fc1_fwd_plain", "fc2_fwd", "fc2_dgrad", "fc1_dgrad", "fc2_wgrad"]
sys.argv = [sys.argv[0], "1", "x"]  # gemm_probe: build the tensors, run nothing
ns = {"__file__": str(ROOT / "tools/gemm_probe.py"), "__name__": "gemm_probe"}
exec(compile(open(ROOT / "tools/gemm_probe.py").read(), "gemm_probe", "exec"), ns)
# the gate GEMM with routing in its epilogue (one 128-row tile per CTA), configs[1] N=1
_ops, _dev = ns["ops"], ns["dev"]
_T, _M, _E, _k = 16384, 1024, 64, 2
_xg = torch.randn(_T, _M, device=_dev).bfloat16()
_wg = torch.randn(_E, _M, device=_dev) / 32
_gout = (torch.empty(_T, _E, device=_dev), torch.empty(_T, _k, device=_dev, dtype=torch.int32),
         torch.empty(_T, _k, device=_dev),
         torch.empty(max(int(_lib.load().mpm_route_workspace_bytes(_T, _E, _k)), 4), device=_dev, dtype=torch.uint8))
_gws = _ops.gate_workspace(_T, _M, _E, _dev)
ns["cases"]["gate_route"] = lambda: _ops.gate_route(_xg, _wg, _k, True, out=_gout, gate_ws=_gws)
# the gate backward GEMMs (dWg = dlogits^T x split-K + reduce; renorm top-2: no dense dx term)
_dl = torch.randn(_T, _E, device=_dev) * 1e-3
_dwg = torch.empty(_E, _M, device=_dev)
_dxg = torch.empty(_T, _M, device=_dev, dtype=torch.bfloat16)
ns["cases"]["gate_bwd"] = lambda: _ops.gate_backward_gemms(_xg, _wg, _dl, _k, True, _dwg, _dxg, _gws)
names = ["prod_wait_empty", "mma_wait_tempty", "mma_wait_full", "epi_wait_tfull", "epi_tmem_ld",
         "epi_wait_stg", "epi_busy", "epi_tiles", "mma_total", "entry_to_pdl", "route_epi", "entry_to_done", "route_tmem", "route_logits_st", "route_topk", "route_counts"]
for name in cases:
    f = ns["cases"][name]
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    fn(buf, 1)
    reps = 5
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    b.synchronize()
    fn(buf, 1)
    v = [buf[i] / reps for i in range(16)]
    ctas = 148
    tiles = v[7] / 4 if v[7] else 1  # per epilogue warp
    out = {"case": name, "us": a.elapsed_time(b) * 1e3 / reps}
    out.update({names[i]: round(v[i]) for i in range(16)})
    # per-tile views: the MMA thread exists on the 74 leader CTAs of the pair kernels
    out["epi_busy_per_warp_tile"] = round(v[6] / v[7]) if v[7] else None
    out["epi_wait_tfull_per_warp_tile"] = round(v[3] / v[7]) if v[7] else None
    out["epi_tmem_ld_per_warp_tile"] = round(v[4] / v[7]) if v[7] else None
    out["epi_wait_stg_per_warp_tile"] = round(v[5] / v[7]) if v[7] else None
    print(json.dumps(out), flush=True)
