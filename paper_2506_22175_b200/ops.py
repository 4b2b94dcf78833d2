"""Typed torch wrappers over the libmpm C-ABI (include/mpm.h).

Each wrapper checks device / dtype / contiguity, passes raw pointers and the
launching stream's cudaStream_t, and raises MpmError on a nonzero status.
PyTorch is plumbing here (device memory, streams); every FLOP and byte of
the MoE data plane moves in libmpm's kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import GemmArgs, call

_DT = {torch.float32: _lib.MPM_F32, torch.bfloat16: _lib.MPM_BF16}


def dtype_code(dt: torch.dtype) -> int:
    if dt not in _DT:
        raise TypeError(f"unsupported dtype {dt}; use torch.float32 or torch.bfloat16")
    return _DT[dt]


def _p(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _s(stream: torch.cuda.Stream | None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need(t: torch.Tensor, name: str, dtype=None, contiguous: bool = True):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if contiguous and not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def capacity(tokens: int, k: int, num_experts: int, capacity_factor: float) -> int:
    """Slots per (source rank, expert): ceil(cf * T * k / E)."""
    import math
    return int(math.ceil(capacity_factor * tokens * k / num_experts - 1e-9))


@dataclass
class Routing:
    logits: torch.Tensor   # [T, E] f32
    idx: torch.Tensor      # [T, k] int32
    weights: torch.Tensor  # [T, k] f32
    slot: torch.Tensor     # [T, k] int32 (-1 dropped)
    kept: torch.Tensor     # [E] int32
    capacity: int
    workspace: torch.Tensor


_WS: dict = {}


def workspace(nbytes: int, device, tag: str = "gate") -> torch.Tensor:
    """Per-(device, tag) scratch reused across calls on one stream order."""
    key = (str(device), tag)
    t = _WS.get(key)
    if t is None or t.numel() < nbytes:
        t = torch.empty(max(nbytes, 256), device=device, dtype=torch.uint8)
        _WS[key] = t
    return t


def gate_workspace(T: int, M: int, E: int, device) -> torch.Tensor:
    return workspace(int(_lib.load().mpm_gate_workspace_bytes(T, M, E)), device, "gate")


def gate_fwd(x: torch.Tensor, wg: torch.Tensor, stream=None, out=None, ws=None) -> torch.Tensor:
    _need(x, "x"); _need(wg, "wg", torch.float32)
    T, M = x.shape
    E = wg.shape[0]
    logits = out if out is not None else torch.empty(T, E, device=x.device, dtype=torch.float32)
    ws = ws if ws is not None else gate_workspace(T, M, E, x.device)
    call("mpm_gate_fwd", _p(x), dtype_code(x.dtype), _p(wg), _p(logits), T, M, E, _p(ws), _s(stream))
    return logits


def route(logits: torch.Tensor, k: int, renorm: bool = True, stream=None, out=None):
    _need(logits, "logits", torch.float32)
    T, E = logits.shape
    if out is None:
        idx = torch.empty(T, k, device=logits.device, dtype=torch.int32)
        w = torch.empty(T, k, device=logits.device, dtype=torch.float32)
        nbytes = _lib.load().mpm_route_workspace_bytes(T, E, k)
        ws = torch.empty(max(nbytes, 4), device=logits.device, dtype=torch.uint8)
    else:
        idx, w, ws = out
    call("mpm_route", _p(logits), T, E, k, int(renorm), _p(idx), _p(w), _p(ws), _s(stream))
    return idx, w, ws


def gate_route(x: torch.Tensor, wg: torch.Tensor, k: int, renorm: bool = True, stream=None, out=None,
               gate_ws=None):
    """Gate GEMM + top-k in one call (`mpm_gate_route`): same results as gate_fwd then route,
    the partial-logit sum folded into the routing kernel.  Returns (logits, idx, weights, route_ws)."""
    _need(x, "x"); _need(wg, "wg", torch.float32)
    T, M = x.shape
    E = wg.shape[0]
    if out is None:
        logits = torch.empty(T, E, device=x.device, dtype=torch.float32)
        idx = torch.empty(T, k, device=x.device, dtype=torch.int32)
        w = torch.empty(T, k, device=x.device, dtype=torch.float32)
        ws = torch.empty(max(_lib.load().mpm_route_workspace_bytes(T, E, k), 4), device=x.device, dtype=torch.uint8)
    else:
        logits, idx, w, ws = out
    gate_ws = gate_ws if gate_ws is not None else gate_workspace(T, M, E, x.device)
    call("mpm_gate_route", _p(x), dtype_code(x.dtype), _p(wg), T, M, E, k, int(renorm), _p(logits), _p(idx), _p(w),
         _p(gate_ws), _p(ws), _s(stream))
    return logits, idx, w, ws


def assign_slots(idx: torch.Tensor, num_experts: int, cap: int, workspace: torch.Tensor, stream=None, out=None):
    _need(idx, "idx", torch.int32)
    T, k = idx.shape
    if out is None:
        slot = torch.empty(T, k, device=idx.device, dtype=torch.int32)
        kept = torch.empty(num_experts, device=idx.device, dtype=torch.int32)
    else:
        slot, kept = out
    call("mpm_assign_slots", _p(idx), T, num_experts, k, cap, _p(workspace), _p(slot), _p(kept), _s(stream))
    return slot, kept


def compute_routing(x: torch.Tensor, wg: torch.Tensor, k: int, cap: int, renorm: bool = True,
                    stream=None, logits: torch.Tensor | None = None) -> Routing:
    if logits is None:
        logits = gate_fwd(x, wg, stream)
    idx, w, ws = route(logits, k, renorm, stream)
    slot, kept = assign_slots(idx, wg.shape[0], cap, ws, stream)
    return Routing(logits, idx, w, slot, kept, cap, ws)


def permute(x: torch.Tensor, r: Routing, n_chunks: int, out: torch.Tensor, stream=None) -> torch.Tensor:
    _need(x, "x"); _need(out, "send", x.dtype)
    T, M = x.shape
    E = r.kept.shape[0]
    k = r.idx.shape[1]
    call("mpm_permute", _p(x), dtype_code(x.dtype), _p(r.idx), _p(r.slot), _p(r.kept), T, M, E, k,
         r.capacity, n_chunks, _p(out), _s(stream))
    return out


def combine(t_o: torch.Tensor, r: Routing, n_chunks: int, T: int, stream=None, out=None) -> torch.Tensor:
    _need(t_o, "t_o")
    M = t_o.shape[-1]
    E = r.kept.shape[0]
    k = r.idx.shape[1]
    y = out if out is not None else torch.empty(T, M, device=t_o.device, dtype=t_o.dtype)
    call("mpm_combine", _p(t_o), dtype_code(t_o.dtype), _p(r.idx), _p(r.slot), _p(r.weights), T, M, E, k,
         r.capacity, n_chunks, _p(y), _s(stream))
    return y


def combine_bwd(dy: torch.Tensor, t_o: torch.Tensor, r: Routing, n_chunks: int, g_o: torch.Tensor | None,
                stream=None, out=None, dprob: bool = True):
    """dprob (returned) and the g_o scatter; g_o=None computes only dprob, dprob=False only g_o."""
    _need(dy, "dy", t_o.dtype); _need(t_o, "t_o")
    if g_o is not None:
        _need(g_o, "g_o", t_o.dtype)
    T, M = dy.shape
    E = r.kept.shape[0]
    k = r.idx.shape[1]
    if dprob:
        dprob = out if out is not None else torch.empty(T, k, device=dy.device, dtype=torch.float32)
    else:
        dprob = None
    call("mpm_combine_bwd", _p(dy), _p(t_o), dtype_code(t_o.dtype), _p(r.idx), _p(r.slot), _p(r.kept),
         _p(r.weights), T, M, E, k, r.capacity, n_chunks, _p(dprob), _p(g_o), _s(stream))
    return dprob


def combine_bwd_gate(dy: torch.Tensor, t_o: torch.Tensor, r: Routing, n_chunks: int, g_o: torch.Tensor | None,
                     dlogits: torch.Tensor, ws: torch.Tensor, renorm: bool = True, dprob: torch.Tensor | None = None,
                     stream=None) -> None:
    """One pass of the combine + gate backward: g_o rows (unless None), dprob (when given), dlogits and
    the split operands of the gate GEMMs in `ws` (mpm_combine_bwd_gate)."""
    _need(dy, "dy", t_o.dtype); _need(t_o, "t_o")
    if g_o is not None:
        _need(g_o, "g_o", t_o.dtype)
    T, M = dy.shape
    E = r.kept.shape[0]
    k = r.idx.shape[1]
    call("mpm_combine_bwd_gate", _p(dy), _p(t_o), dtype_code(t_o.dtype), _p(r.idx), _p(r.slot), _p(r.kept),
         _p(r.weights), _p(r.logits), T, M, E, k, int(renorm), r.capacity, n_chunks, _p(g_o), _p(dprob),
         _p(dlogits), _p(ws), _s(stream))


def gate_backward_gemms(x: torch.Tensor, wg: torch.Tensor, dlogits: torch.Tensor, k: int, renorm: bool,
                        dwg: torch.Tensor, dx: torch.Tensor, ws: torch.Tensor, stream=None) -> None:
    """dwg = dlogits^T x and, for the dense gate gradient, the gate term of dx (mpm_gate_backward_gemms)."""
    T, M = x.shape
    E = dlogits.shape[1]
    call("mpm_gate_backward_gemms", _p(x), dtype_code(x.dtype), _p(wg), _p(dlogits), T, M, E, k, int(renorm),
         _p(dwg), _p(dx), _p(ws), _s(stream))


def gate_gather(r: Routing, g_i: torch.Tensor, wg: torch.Tensor, n_chunks: int, dlogits: torch.Tensor,
                renorm: bool, dx: torch.Tensor, ws: torch.Tensor, stream=None) -> torch.Tensor:
    """dx = gathered g_i rows + the gate term (mpm_gate_gather)."""
    T, M = dx.shape
    E = r.kept.shape[0]
    k = r.idx.shape[1]
    call("mpm_gate_gather", _p(g_i), dtype_code(dx.dtype), _p(r.idx), _p(r.slot), _p(dlogits), _p(wg), T, M, E,
         k, int(renorm), r.capacity, n_chunks, _p(dx), _p(ws), _s(stream))
    return dx


def gate_bwd_logits(r: Routing, dprob: torch.Tensor, renorm: bool = True, stream=None, out=None) -> torch.Tensor:
    T, E = r.logits.shape
    k = r.idx.shape[1]
    dl = out if out is not None else torch.empty(T, E, device=dprob.device, dtype=torch.float32)
    call("mpm_gate_bwd_logits", _p(r.logits), _p(r.idx), _p(r.weights), _p(dprob), T, E, k, int(renorm),
         _p(dl), _s(stream))
    return dl


def gather_bwd(g_i: torch.Tensor, r: Routing, dlogits: torch.Tensor, wg: torch.Tensor, n_chunks: int,
               T: int, stream=None) -> torch.Tensor:
    _need(g_i, "g_i"); _need(wg, "wg", torch.float32)
    M = g_i.shape[-1]
    E = r.kept.shape[0]
    k = r.idx.shape[1]
    dx = torch.empty(T, M, device=g_i.device, dtype=g_i.dtype)
    ws = gate_workspace(T, M, E, g_i.device)
    call("mpm_gather_bwd", _p(g_i), dtype_code(g_i.dtype), _p(r.idx), _p(r.slot), _p(dlogits), _p(wg),
         T, M, E, k, r.capacity, n_chunks, _p(dx), _p(ws), _s(stream))
    return dx


def gate_backward(r: Routing, dprob: torch.Tensor, x: torch.Tensor, g_i: torch.Tensor, wg: torch.Tensor,
                  n_chunks: int, renorm: bool = True, stream=None, dlogits=None, ws=None):
    """Fused gate backward: (dx, dwg, dlogits)."""
    T, M = x.shape
    E = r.kept.shape[0]
    k = r.idx.shape[1]
    dl = dlogits if dlogits is not None else torch.empty(T, E, device=x.device, dtype=torch.float32)
    dx = torch.empty(T, M, device=x.device, dtype=x.dtype)
    dwg = torch.empty(E, M, device=x.device, dtype=torch.float32)
    ws = ws if ws is not None else gate_workspace(T, M, E, x.device)
    call("mpm_gate_backward", _p(r.logits), _p(r.idx), _p(r.weights), _p(dprob), _p(x), _p(g_i), _p(r.slot),
         dtype_code(x.dtype), _p(wg), T, M, E, k, int(renorm), r.capacity, n_chunks, _p(dl), _p(dx), _p(dwg),
         _p(ws), _s(stream))
    return dx, dwg, dl


def gate_backward_gate(r: Routing, dprob: torch.Tensor, x: torch.Tensor, wg: torch.Tensor, renorm: bool = True,
                       stream=None, dlogits=None, dwg=None, ws=None, dx=None):
    """First half of gate_backward (no expert-side input): (dwg, dlogits, dx); on the
    tcgen05 path dx already holds the gate term dl.wg (pass the same dx to the gather)."""
    T, M = x.shape
    E = r.kept.shape[0]
    k = r.idx.shape[1]
    dl = dlogits if dlogits is not None else torch.empty(T, E, device=x.device, dtype=torch.float32)
    dwg = dwg if dwg is not None else torch.empty(E, M, device=x.device, dtype=torch.float32)
    dx = dx if dx is not None else torch.empty(T, M, device=x.device, dtype=x.dtype)
    call("mpm_gate_backward_gate", _p(r.logits), _p(r.idx), _p(r.weights), _p(dprob), _p(x), dtype_code(x.dtype),
         _p(wg), T, M, E, k, int(renorm), _p(dl), _p(dwg), _p(dx), _p(ws), _s(stream))
    return dwg, dl, dx


def gate_backward_gather(r: Routing, g_i: torch.Tensor, x: torch.Tensor, wg: torch.Tensor, n_chunks: int,
                         dlogits: torch.Tensor, ws: torch.Tensor, dx: torch.Tensor, stream=None) -> torch.Tensor:
    """Second half of gate_backward: dx += gathered g_i rows (dx from gate_backward_gate)."""
    T, M = x.shape
    E = r.kept.shape[0]
    call("mpm_gate_backward_gather", _p(g_i), dtype_code(x.dtype), _p(r.idx), _p(r.slot), _p(dlogits), _p(wg),
         T, M, E, r.idx.shape[1], r.capacity, n_chunks, _p(dx), _p(ws), _s(stream))
    return dx


def gate_wgrad(dlogits: torch.Tensor, x: torch.Tensor, stream=None, out=None) -> torch.Tensor:
    T, M = x.shape
    E = dlogits.shape[1]
    dwg = out if out is not None else torch.empty(E, M, device=x.device, dtype=torch.float32)
    ws = gate_workspace(T, M, E, x.device)
    call("mpm_gate_wgrad", _p(dlogits), _p(x), dtype_code(x.dtype), T, M, E, _p(dwg), _p(ws), _s(stream))
    return dwg


def gemm(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, *, a_mn_major: bool = False,
         b_mn_major: bool = False, epilogue: int = _lib.EPI_NONE, aux: torch.Tensor | None = None,
         valid_rows: torch.Tensor | None = None, valid_k: torch.Tensor | None = None, stream=None,
         simt: bool = False,
         k_splits: int = 1, split_stride: int = 0, a_k_period: int = 0, b_k_period: int = 0,
         k: int | None = None) -> torch.Tensor:
    """Batched C[b] = A[b] . B[b]^T on 3-D (batch, ., .) views with unit inner stride.

    a: [B, rows, K] (a_mn_major=False) or [B, K, rows] (True)
    b: [B, N, K]    (b_mn_major=False) or [B, K, N]    (True)
    c: [B, rows, N]
    """
    for t, name in ((a, "a"), (b, "b"), (c, "c")):
        if t.dim() != 3 or t.stride(2) != 1 or not t.is_cuda:
            raise ValueError(f"{name} must be a 3-D CUDA view with unit inner stride")
    if a.dtype != b.dtype:
        raise TypeError("a and b must share a dtype")
    batches = a.shape[0]
    rows, K = (a.shape[2], a.shape[1]) if a_mn_major else (a.shape[1], a.shape[2])
    N = b.shape[2] if b_mn_major else b.shape[1]
    if k is not None:  # logical K of K-periodic operands
        K = k
    if k_splits <= 1 and tuple(c.shape) != (batches, rows, N):
        raise ValueError(f"c shape {tuple(c.shape)} != {(batches, rows, N)}")
    args = GemmArgs()
    args.dtype = dtype_code(a.dtype)
    args.epilogue = epilogue
    args.batches, args.rows, args.n, args.k = batches, rows, N, K
    args.a, args.a_ld, args.a_batch_stride, args.a_mn_major = a.data_ptr(), a.stride(1), a.stride(0), int(a_mn_major)
    args.b, args.b_ld, args.b_batch_stride, args.b_mn_major = b.data_ptr(), b.stride(1), b.stride(0), int(b_mn_major)
    args.c, args.c_ld, args.c_batch_stride, args.c_dtype = c.data_ptr(), c.stride(1), c.stride(0), dtype_code(c.dtype)
    if aux is not None:
        args.aux, args.aux_ld, args.aux_batch_stride = aux.data_ptr(), aux.stride(1), aux.stride(0)
    if valid_rows is not None:
        _need(valid_rows, "valid_rows", torch.int32)
        args.valid_rows = valid_rows.data_ptr()
    if valid_k is not None:
        _need(valid_k, "valid_k", torch.int32)
        args.valid_k = valid_k.data_ptr()
    args.a_k_period, args.b_k_period = a_k_period, b_k_period
    args.k_splits, args.split_stride = k_splits, split_stride
    call("mpm_grouped_gemm_simt" if simt else "mpm_grouped_gemm", ctypes.byref(args), _s(stream))
    return c


def splitk_reduce(partials: torch.Tensor, splits: int, split_stride: int, out: torch.Tensor,
                  accumulate: bool = False, stream=None) -> torch.Tensor:
    call("mpm_splitk_reduce", _p(partials), splits, split_stride, out.numel(), _p(out), dtype_code(out.dtype),
         int(accumulate), _s(stream))
    return out


def copy_async(dst: torch.Tensor, src: torch.Tensor, stream=None) -> None:
    if dst.numel() != src.numel() or dst.dtype != src.dtype:
        raise ValueError("copy_async: size/dtype mismatch")
    if src.is_cuda and not dst.is_cuda:
        direction = _lib.COPY_D2H
    elif dst.is_cuda and not src.is_cuda:
        direction = _lib.COPY_H2D
    else:
        direction = _lib.COPY_D2D
    nbytes = src.numel() * src.element_size()
    call("mpm_copy_async", _p(dst), _p(src), nbytes, direction, _s(stream))


def sm_count() -> int:
    return int(_lib.load().mpm_sm_count())
