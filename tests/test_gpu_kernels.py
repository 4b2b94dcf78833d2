"""Kernel-level parity of libmpm against the CPU oracle / a torch fp32 reference.

Bars (north star): routing indices, expert assignment and capacity drops
bit-exact; fp32 rtol 1e-5; bf16 rtol 2e-2 against an fp32 reference.
Every tolerance below is |got - ref| <= rtol*|ref| + atol with the atol
stated at the call site (scale-relative for near-zero entries).
"""

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from paper_2506_22175_b200 import _lib, ops

pytestmark = pytest.mark.gpu


def _close(got, ref, rtol, atol_scale=None):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    atol = (atol_scale if atol_scale is not None else rtol) * max(np.abs(ref).max(), 1e-30)
    err = np.abs(got - ref) - (rtol * np.abs(ref) + atol)
    assert err.max() <= 0, f"max violation {err.max():.3e} (rtol {rtol}, atol {atol:.3e})"


@pytest.mark.parametrize("T,E,k,renorm", [(2048, 4, 1, True), (4096, 64, 2, True), (3000, 128, 1, True),
                                          (1000, 16, 4, False), (513, 8, 2, True), (1, 4, 1, True),
                                          (777, 32, 8, True), (300, 8, 8, False), (2048, 256, 6, True),
                                          (1001, 24, 3, True), (96, 12, 5, False)])
def test_route_and_slots_bitexact(cuda, T, E, k, renorm):
    rng = np.random.default_rng(T * 31 + E)
    logits = rng.standard_normal((T, E)).astype(np.float32)
    logits[::7] = np.round(logits[::7] * 4) / 4  # exact ties exercise the lowest-index rule
    lg = torch.from_numpy(logits).to(cuda)
    C = O.capacity(T, k, E, 1.0)
    r = ops.compute_routing(None, torch.zeros(E, 8, device=cuda), k, C, renorm, logits=lg)
    idx_ref, w_ref = O.route(logits, k, renorm)
    slot_ref, kept_ref = O.assign_slots(idx_ref, E, C)
    np.testing.assert_array_equal(r.idx.cpu().numpy(), idx_ref)
    np.testing.assert_array_equal(r.slot.cpu().numpy(), slot_ref)
    np.testing.assert_array_equal(r.kept.cpu().numpy(), kept_ref)
    _close(r.weights.cpu().numpy(), w_ref, 1e-5, 0)
    assert ops.capacity(T, k, E, 1.0) == C


def test_skewed_routing_drops_bitexact(cuda):
    T, E, k = 8192, 32, 2
    rng = np.random.default_rng(5)
    logits = rng.standard_normal((T, E)).astype(np.float32)
    logits[:, : E // 4] += 2.0  # +2 logit bias on 25% of experts -> heavy drops
    C = O.capacity(T, k, E, 1.0)
    r = ops.compute_routing(None, torch.zeros(E, 8, device=cuda), k, C, True,
                            logits=torch.from_numpy(logits).to(cuda))
    idx_ref, _ = O.route(logits, k, True)
    slot_ref, kept_ref = O.assign_slots_fast(idx_ref, E, C)
    assert (slot_ref < 0).sum() > 0
    np.testing.assert_array_equal(r.slot.cpu().numpy(), slot_ref)
    np.testing.assert_array_equal(r.kept.cpu().numpy(), kept_ref)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("E", [64, 8, 6, 40])  # E % 32 != 0: expert axis zero-padded on the tensor-core path
def test_gate_logits(cuda, dtype, E):
    T, M = 1000, 512
    g = torch.Generator().manual_seed(1)
    x = torch.randn(T, M, generator=g).to(dtype)
    wg = torch.randn(E, M, generator=g) / M ** 0.5
    got = ops.gate_fwd(x.to(cuda), wg.to(cuda)).cpu().numpy()
    ref = O.gate_logits(x.float().numpy(), wg.numpy())
    _close(got, ref, 1e-5, 1e-6)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("T,M,E,k,renorm", [(1000, 512, 64, 2, True), (4096, 1024, 128, 1, True),
                                            (333, 256, 32, 4, False), (1, 64, 8, 1, True), (77, 48, 6, 2, True),
                                            (40000, 256, 64, 2, True), (40000, 128, 40, 1, True),
                                            (512, 128, 64, 8, True), (700, 256, 64, 3, False)])
def test_gate_route_fused_matches_two_calls(cuda, dtype, T, M, E, k, renorm):
    """mpm_gate_route is bit-identical to mpm_gate_fwd + mpm_route: logits, indices, weights and the
    per-block counts.  On the tensor-core path with E <= 64 the routing runs in the gate GEMM's
    epilogue (single-CTA tiles, and 2-CTA pair tiles from ~38K tokens on: T = 40000); E = 128 sums the
    stored partial logits in the routing kernel."""
    g = torch.Generator().manual_seed(T + E)
    x = torch.randn(T, M, generator=g).to(dtype).to(cuda)
    wg = (torch.randn(E, M, generator=g) / M ** 0.5).to(cuda)
    logits, idx, w, ws = ops.gate_route(x, wg, k, renorm)
    ref_logits = ops.gate_fwd(x, wg)
    ref_idx, ref_w, ref_ws = ops.route(ref_logits, k, renorm)
    assert torch.equal(logits, ref_logits)
    assert torch.equal(idx, ref_idx)
    assert torch.equal(w, ref_w)
    half = ws.numel() // 2  # [k][nblk][E] counts; the second half is assign_slots scratch
    assert torch.equal(ws[:half], ref_ws[:half])
    idx_o, _ = O.route(ref_logits.cpu().numpy(), k, renorm)
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_o)


@pytest.mark.parametrize("T,M,E", [(300, 256, 64), (300, 256, 8), (512, 256, 6), (1000, 512, 40)])
def test_gate_partials_fully_written(cuda, T, M, E):
    """Every partial logit the routing kernel reads is written by the gate GEMM: a NaN-filled
    workspace leaves no NaN in the logits (and none in the [T][3Ec] partials themselves)."""
    x = torch.randn(T, M, device=cuda).bfloat16()
    wg = torch.randn(E, M, device=cuda) / 16
    ws = ops.gate_workspace(T, M, E, cuda)
    ws.view(torch.uint8).fill_(0xFF)  # all-ones bytes: NaN as f32
    logits, idx, w, _ = ops.gate_route(x, wg, 2, gate_ws=ws)  # E <= 64: routed in the GEMM epilogue
    assert not torch.isnan(logits).any() and not torch.isnan(w).any()
    ws.view(torch.uint8).fill_(0xFF)
    logits = ops.gate_fwd(x, wg, ws=ws)  # stores the partials, then sums them
    assert not torch.isnan(logits).any()
    Ec, Mp = -(-E // 32) * 32, -(-M // 64) * 64
    off = (Ec * 3 * Mp * 2 + 255) // 256 * 256
    part = ws[off:off + T * 3 * Ec * 4].view(torch.float32).view(T, 3 * Ec)
    assert not torch.isnan(part).any()
    assert torch.equal(part[:, E:Ec], torch.zeros_like(part[:, E:Ec]))  # zero-padded experts


@pytest.mark.parametrize("n", [1, 3])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_permute_layout_and_combine(cuda, n, dtype):
    T, M, E, k = 777, 64, 8, 2
    g = torch.Generator().manual_seed(2)
    x = torch.randn(T, M, generator=g).to(dtype)
    wg = torch.randn(E, M, generator=g)
    C = O.capacity(T, k, E, 1.0)
    xd = x.to(cuda)
    r = ops.compute_routing(xd, wg.to(cuda), k, C, True)
    send = torch.full((E * C, M), float("nan"), device=cuda, dtype=dtype)
    ops.permute(xd, r, n, send)
    idx, slot = r.idx.cpu().numpy(), r.slot.cpu().numpy()
    ref = np.zeros((E * C, M), dtype=np.float32)
    row = lambda e, s: e * C + s  # expert-major slot layout (include/mpm.h)
    for t in range(T):
        for j in range(k):
            if slot[t, j] >= 0:
                ref[row(idx[t, j], slot[t, j])] = x[t].float().numpy()
    np.testing.assert_array_equal(send.float().cpu().numpy(), ref)  # zero-filled padding, exact copy
    # combine: y = sum_j w_j * t_o[row_j] with t_o = send (identity experts)
    y = ops.combine(send, r, n, T).float().cpu().numpy()
    w = r.weights.cpu().numpy()
    y_ref = np.zeros((T, M))
    for j in range(k):
        keep = slot[:, j] >= 0
        y_ref[keep] += w[keep, j:j + 1] * x.float().numpy()[keep]
    _close(y, y_ref, 1e-5 if dtype == torch.float32 else 1e-2, 1e-6 if dtype == torch.float32 else 1e-2)


def _ref_gemm(a, b, a_mn, b_mn):
    A = a.float().transpose(1, 2) if a_mn else a.float()
    B = b.float().transpose(1, 2) if b_mn else b.float()
    return torch.bmm(A.double(), B.double().transpose(1, 2))


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("rows,N,K", [(128, 256, 64), (300, 512, 200), (77, 96, 1000), (512, 1024, 4096)])
def test_tcgen05_gemm_layouts(cuda, a_mn, b_mn, rows, N, K):
    B = 3
    g = torch.Generator(device=cuda).manual_seed(rows + N + K)
    pad = lambda v: (v + 7) // 8 * 8  # TMA: 16-byte aligned pitches; logical extents stay ragged
    a = torch.randn((B, K, pad(rows)) if a_mn else (B, rows, pad(K)), device=cuda, generator=g).bfloat16()
    a = a[:, :, :rows] if a_mn else a[:, :, :K]
    b = torch.randn((B, K, N) if b_mn else (B, N, pad(K)), device=cuda, generator=g).bfloat16()
    b = b if b_mn else b[:, :, :K]
    c = torch.full((B, rows, N), float("nan"), device=cuda, dtype=torch.float32)
    ops.gemm(a, b, c, a_mn_major=a_mn, b_mn_major=b_mn, epilogue=_lib.EPI_STORE_F32)
    ref = _ref_gemm(a, b, a_mn, b_mn)
    # bf16 operands, fp32 accumulation: differences come from summation order only
    _close(c.cpu().numpy(), ref.cpu().numpy(), 1e-4, 1e-4)


@pytest.mark.parametrize("epi", ["relu", "drelu", "accum", "accum_bf16", "accum_f32_generic", "add_aux",
                                 "store_bf16", "relu_mask", "dmask"])
def test_tcgen05_epilogues(cuda, epi):
    B, rows, N, K = 2, 200, 256, 256
    g = torch.Generator(device=cuda).manual_seed(9)
    a = torch.randn(B, rows, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(B, N, K, device=cuda, generator=g).bfloat16()
    acc = _ref_gemm(a, b, False, False)
    aux_bf = torch.randn(B, rows, N, device=cuda, generator=g).bfloat16()
    base = torch.randn(B, rows, N, device=cuda, generator=g)
    if epi == "relu":
        c = torch.empty(B, rows, N, device=cuda, dtype=torch.bfloat16)
        ops.gemm(a, b, c, epilogue=_lib.EPI_RELU)
        ref = acc.clamp_min(0)
    elif epi == "drelu":
        c = torch.empty(B, rows, N, device=cuda, dtype=torch.bfloat16)
        ops.gemm(a, b, c, epilogue=_lib.EPI_DRELU, aux=aux_bf)
        ref = acc * (aux_bf.float() > 0)
    elif epi == "accum":
        c = base.clone()
        ops.gemm(a, b, c, epilogue=_lib.EPI_ACCUM_F32)
        ref = acc + base.double()
    elif epi == "accum_bf16":  # in-place bf16 wgrad accumulation (TMA reduce-add, bf16 tensor map)
        c = base.bfloat16()
        ops.gemm(a, b, c, epilogue=_lib.EPI_ACCUM)
        ref = acc + base.bfloat16().double()
    elif epi == "accum_f32_generic":
        c = base.clone()
        ops.gemm(a, b, c, epilogue=_lib.EPI_ACCUM)
        ref = acc + base.double()
    elif epi == "add_aux":
        c = torch.empty(B, rows, N, device=cuda, dtype=torch.bfloat16)
        ops.gemm(a, b, c, epilogue=_lib.EPI_ADD_AUX_F32, aux=base)
        ref = acc + base.double()
    elif epi == "store_bf16":
        c = torch.empty(B, rows, N, device=cuda, dtype=torch.bfloat16)
        ops.gemm(a, b, c)
        ref = acc
    elif epi == "relu_mask":
        c = torch.empty(B, rows, N, device=cuda, dtype=torch.bfloat16)
        mask = torch.full((B, rows, N // 32), -1, device=cuda, dtype=torch.int32)
        ops.gemm(a, b, c, epilogue=_lib.EPI_RELU_MASK, aux=mask)
        ref = acc.clamp_min(0)
        bits = ((mask.cpu().numpy().astype(np.int64)[..., None] >> np.arange(32)) & 1).reshape(B, rows, N)
        np.testing.assert_array_equal(bits, (acc > 0).cpu().numpy().astype(np.int64))
    else:  # dmask: multiply by the bits of a random mask
        c = torch.empty(B, rows, N, device=cuda, dtype=torch.bfloat16)
        mask = torch.randint(-2**31, 2**31 - 1, (B, rows, N // 32), device=cuda, dtype=torch.int32)
        ops.gemm(a, b, c, epilogue=_lib.EPI_DMASK, aux=mask)
        bits = ((mask.cpu().numpy().astype(np.int64)[..., None] >> np.arange(32)) & 1).reshape(B, rows, N)
        ref = acc * torch.from_numpy(bits).to(cuda)
    tol = 1e-4 if c.dtype == torch.float32 else 8e-3
    _close(c.float().cpu().numpy(), ref.cpu().numpy(), tol, tol)


def test_simt_gemm_fp32_exactish(cuda):
    B, rows, N, K = 2, 100, 70, 300
    g = torch.Generator(device=cuda).manual_seed(4)
    a = torch.randn(B, K, rows, device=cuda, generator=g)
    b = torch.randn(B, K, N, device=cuda, generator=g)
    c = torch.empty(B, rows, N, device=cuda)
    with pytest.raises(_lib.MpmError):  # N % 32 != 0 has no tcgen05 path: loud error, not a fallback
        ops.gemm(a.bfloat16(), b.bfloat16(), c, a_mn_major=True, b_mn_major=True, epilogue=_lib.EPI_STORE_F32)
    ops.gemm(a, b, c, a_mn_major=True, b_mn_major=True)
    _close(c.cpu().numpy(), _ref_gemm(a, b, True, True).cpu().numpy(), 1e-5, 1e-6)


@pytest.mark.parametrize("T,M,E", [(1024, 512, 64), (1000, 256, 64), (4096, 1024, 128), (2048, 256, 4),
                                   (16384, 1024, 8)])
def test_gate_backward_kernels(cuda, T, M, E):
    """dWg = dl^T x (tcgen05 bf16x3 split-K when T % 64 == 0) and dx = dl Wg + gathered rows."""
    g = torch.Generator().manual_seed(T + E)
    x = torch.randn(T, M, generator=g).bfloat16()
    dl = torch.randn(T, E, generator=g) * 1e-2
    wg = torch.randn(E, M, generator=g) / M ** 0.5
    dwg = ops.gate_wgrad(dl.to(cuda), x.to(cuda)).cpu().double().numpy()
    ref = dl.double().numpy().T @ x.double().numpy()
    _close(dwg, ref, 1e-5, 1e-6)
    # gather: identity routing rows (k=1, C=T/E...) exercised through a tiny routing of T tokens
    k = 2
    C = O.capacity(T, k, E, 1.0)
    r = ops.compute_routing(x.to(cuda), wg.to(cuda), k, C, True)
    g_i = torch.randn(E * C, M, generator=g).bfloat16().to(cuda)
    dx = ops.gather_bwd(g_i, r, dl.to(cuda), wg.to(cuda), 1, T).float().cpu().numpy()
    idx, slot = r.idx.cpu().numpy(), r.slot.cpu().numpy()
    gi = g_i.float().cpu().numpy()
    dx_ref = dl.double().numpy() @ wg.double().numpy()
    for j in range(k):
        keep = slot[:, j] >= 0
        dx_ref[keep] += gi[idx[keep, j] * C + slot[keep, j]]
    _close(dx, dx_ref, 1e-2, 1e-2)  # bf16 output


def test_splitk_and_k_period(cuda):
    g = torch.Generator(device=cuda).manual_seed(11)
    B, rows, N, K = 1, 128, 512, 4096
    a = torch.randn(B, rows, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(B, N, K, device=cuda, generator=g).bfloat16()
    splits = 7
    part = torch.full((splits, rows, N), float("nan"), device=cuda)
    ops.gemm(a, b, part.view(splits * 1, rows, N)[0:1], epilogue=_lib.EPI_STORE_F32, k_splits=splits,
             split_stride=rows * N)
    out = torch.empty(rows, N, device=cuda)
    kb = (K + 63) // 64
    per = -(-kb // splits)
    ops.splitk_reduce(part, -(-kb // per), rows * N, out)
    _close(out.cpu().numpy(), _ref_gemm(a, b, False, False)[0].cpu().numpy(), 1e-4, 1e-4)
    # K-periodic A: logical K = 3*K0 reads a's K0 columns three times
    K0 = 256
    a0 = a[:, :, :K0].contiguous()
    bb = torch.randn(B, N, 3 * K0, device=cuda, generator=g).bfloat16()
    c = torch.empty(B, rows, N, device=cuda)
    ops.gemm(a0, bb, c, epilogue=_lib.EPI_STORE_F32, a_k_period=K0, k=3 * K0)
    ref = _ref_gemm(a0.repeat(1, 1, 3), bb, False, False)
    _close(c.cpu().numpy(), ref.cpu().numpy(), 1e-4, 1e-4)


def test_simt_split_k_fixed_order(cuda):
    """Exact-fp32 FMA GEMM with K split over blocks: partials per split, summed in split order."""
    g = torch.Generator(device=cuda).manual_seed(12)
    rows, N, K, splits = 8, 200, 5000, 9
    a = torch.randn(1, K, rows, device=cuda, generator=g)       # MN-major, like dlogits^T
    b = torch.randn(1, K, N, device=cuda, generator=g)
    part = torch.full((splits, rows, N), float("nan"), device=cuda)
    ops.gemm(a, b, part[0:1], a_mn_major=True, b_mn_major=True, simt=True, epilogue=_lib.EPI_STORE_F32,
             k_splits=splits, split_stride=rows * N)
    out = torch.empty(rows, N, device=cuda)
    ops.splitk_reduce(part, splits, rows * N, out)
    ref = _ref_gemm(a, b, True, True)[0]
    _close(out.cpu().numpy(), ref.cpu().numpy(), 1e-5, 1e-6)
    per = -(-K // splits)  # each partial is the plain sum over its own K range
    ref0 = _ref_gemm(a[:, :per], b[:, :per], True, True)[0]
    _close(part[0].cpu().numpy(), ref0.cpu().numpy(), 1e-5, 1e-6)
    with pytest.raises(_lib.MpmError):  # split-K writes f32 partials only
        ops.gemm(a, b, part[0:1].bfloat16(), a_mn_major=True, b_mn_major=True, simt=True, k_splits=splits,
                 split_stride=rows * N)


@pytest.mark.parametrize("N", [64, 128, 96, 160, 192])
def test_narrow_n_tiles(cuda, N):
    """N tiles narrower than 256 (64 / 128 wide, and partial 256-wide tiles: 160, 192 = the gate's three
    stacked 64-expert terms), every operand layout and the bf16 (64-column TMA store) output."""
    g = torch.Generator(device=cuda).manual_seed(N)
    for a_mn, b_mn in ((False, False), (True, True), (False, True), (True, False)):
        a = torch.randn((2, 512, 304) if a_mn else (2, 300, 512), device=cuda, generator=g).bfloat16()
        a = a[:, :, :300] if a_mn else a
        b = torch.randn((2, 512, N) if b_mn else (2, N, 512), device=cuda, generator=g).bfloat16()
        c = torch.empty(2, 300, N, device=cuda)
        ops.gemm(a, b, c, a_mn_major=a_mn, b_mn_major=b_mn, epilogue=_lib.EPI_STORE_F32)
        ref = _ref_gemm(a, b, a_mn, b_mn).cpu().numpy()
        _close(c.cpu().numpy(), ref, 1e-4, 1e-4)
        cb = torch.empty(2, 300, N, device=cuda, dtype=torch.bfloat16)
        ops.gemm(a, b, cb, a_mn_major=a_mn, b_mn_major=b_mn)
        _close(cb.float().cpu().numpy(), ref, 1e-2, 1e-2)


def test_launch_counter_counts_kernels(cuda):
    n0 = _lib.launch_count()
    x = torch.randn(256, 64, device=cuda).bfloat16()
    ops.compute_routing(x, torch.randn(8, 64, device=cuda), 2, 64, True)
    assert _lib.launch_count() - n0 >= 4  # gate (split+gemm or simt), route, scan, slot


def test_nccl_grouped_send_recv_single_rank(cuda):
    """The NCCL path of mpm_a2a_chunk (grouped send/recv per block) on a 1-rank communicator,
    with a non-trivial block permutation (the N>1 code path, minus the peers)."""
    import ctypes
    uid = (ctypes.c_char * 128)()
    _lib.call("mpm_comm_unique_id", ctypes.cast(uid, ctypes.c_void_p))
    comm = ctypes.c_void_p()
    _lib.call("mpm_comm_init", ctypes.cast(uid, ctypes.c_void_p), 1, 0, 0, ctypes.byref(comm))
    try:
        blocks, blk = 4, 1024
        src = torch.arange(blocks * blk, device=cuda, dtype=torch.float32).bfloat16()
        dst = torch.full_like(src, -1)
        perm = [2, 0, 3, 1]
        n = blocks
        _lib.call("mpm_a2a_chunk", comm, 1, n, (ctypes.c_int32 * n)(*[0] * n),
                  (ctypes.c_int64 * n)(*[b * blk for b in range(n)]),
                  (ctypes.c_int64 * n)(*[perm[b] * blk for b in range(n)]), blk, _lib.MPM_BF16,
                  ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        for b in range(n):
            assert torch.equal(dst[perm[b] * blk:(perm[b] + 1) * blk], src[b * blk:(b + 1) * blk])
    finally:
        _lib.call("mpm_comm_destroy", comm)


@pytest.mark.parametrize("T,M,E,k,renorm", [(2048, 512, 64, 2, True), (1024, 256, 32, 1, True),
                                            (1000, 256, 16, 2, False), (4096, 512, 8, 2, True),
                                            (1024, 256, 6, 1, True), (2048, 256, 40, 4, False)])
def test_fused_gate_backward_matches_oracle(cuda, T, M, E, k, renorm):
    """mpm_gate_backward (dlogits + dWg + dx in one call) against the oracle's gate gradient."""
    g = torch.Generator().manual_seed(T + M)
    x = torch.randn(T, M, generator=g).bfloat16()
    wg = torch.randn(E, M, generator=g) / M ** 0.5
    C = O.capacity(T, k, E, 1.0)
    r = ops.compute_routing(x.to(cuda), wg.to(cuda), k, C, renorm)
    dprob = (torch.randn(T, k, generator=g) * 0.1).to(cuda)
    g_i = torch.randn(E * C, M, generator=g).bfloat16().to(cuda)
    dx, dwg, dl = ops.gate_backward(r, dprob, x.to(cuda), g_i, wg.to(cuda), 1, renorm)
    idx, w, slot = r.idx.cpu().numpy(), r.weights.cpu().numpy(), r.slot.cpu().numpy()
    dl_ref = O.gate_grad(r.logits.cpu().numpy(), idx, w, dprob.cpu().numpy(), renorm)
    _close(dl.cpu().numpy(), dl_ref, 1e-5, 1e-6)
    _close(dwg.cpu().numpy(), dl_ref.T @ x.double().numpy(), 1e-4, 1e-5)
    dx_ref = dl_ref @ wg.double().numpy()
    gi = g_i.float().cpu().numpy()
    for j in range(k):
        keep = slot[:, j] >= 0
        dx_ref[keep] += gi[idx[keep, j] * C + slot[keep, j]]
    _close(dx.float().cpu().numpy(), dx_ref, 1e-2, 1e-2)
    # the split halves (gate part on a side stream, gather after it) give the fused call's bits
    ws = ops.gate_workspace(T, M, E, cuda)
    side = torch.cuda.Stream(device=cuda)
    side.wait_stream(torch.cuda.current_stream())
    dwg2, dl2, dx2 = ops.gate_backward_gate(r, dprob, x.to(cuda), wg.to(cuda), renorm, stream=side, ws=ws)
    torch.cuda.current_stream().wait_stream(side)
    ops.gate_backward_gather(r, g_i, x.to(cuda), wg.to(cuda), 1, dl2, ws, dx2)
    torch.cuda.synchronize()
    assert torch.equal(dl2, dl) and torch.equal(dwg2, dwg) and torch.equal(dx2, dx)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_combine_bwd_halves_match_fused(cuda, k):
    """combine_bwd with only the dprob half and only the g_o half gives the fused call's bits."""
    T, M, E = 1500, 256, 16
    g = torch.Generator(device=cuda).manual_seed(k)
    x = torch.randn(T, M, device=cuda, generator=g).bfloat16()
    wg = torch.randn(E, M, device=cuda, generator=g) / 16
    C = ops.capacity(T, k, E, 0.8)  # drops on
    r = ops.compute_routing(x, wg, k, C, True)
    t_o = torch.randn(E * C, M, device=cuda, generator=g).bfloat16()
    dy = torch.randn(T, M, device=cuda, generator=g).bfloat16()
    g_o = torch.full((E * C, M), float("nan"), device=cuda, dtype=torch.bfloat16)
    dprob = ops.combine_bwd(dy, t_o, r, 2, g_o)
    g_o2 = torch.full_like(g_o, float("nan"))
    assert ops.combine_bwd(dy, t_o, r, 2, g_o2, dprob=False) is None
    dprob2 = ops.combine_bwd(dy, t_o, r, 2, None)
    torch.cuda.synchronize()
    assert torch.equal(dprob, dprob2)
    assert torch.equal(g_o, g_o2)


@pytest.mark.parametrize("simt", [False, True])
@pytest.mark.parametrize("epi", ["store_f32", "store_bf16", "accum_bf16"])
def test_valid_rows_and_valid_k(cuda, simt, epi):
    """Capacity-padding skip: per-batch valid_k stops the K loop at the covering 64-block (the
    operands' rows beyond it are never read: NaN there must not leak), valid_k = 0 writes zeros,
    and valid_rows leaves the output rows of all-padding tiles untouched."""
    B, rows, N, K = 4, 256, 256, 512
    g = torch.Generator(device=cuda).manual_seed(5)
    # weight-gradient layout: A [b][K][rows], B [b][K][N] (MN-major), K = capacity rows
    a = torch.randn(B, K, rows, device=cuda, generator=g).bfloat16()
    b = torch.randn(B, K, N, device=cuda, generator=g).bfloat16()
    vk = torch.tensor([512, 300, 0, 64], device=cuda, dtype=torch.int32)
    for e in range(B):  # padding rows: zero up to the 64 boundary, NaN beyond (never read)
        cov = -(-int(vk[e]) // 64) * 64
        a[e, int(vk[e]):cov] = 0
        b[e, int(vk[e]):cov] = 0
        a[e, cov:] = float("nan")
        b[e, cov:] = float("nan")
    dt = torch.float32 if epi == "store_f32" else torch.bfloat16
    c = torch.randn(B, rows, N, device=cuda, generator=g).to(dt)
    c0 = c.clone()
    code = {"store_f32": _lib.EPI_STORE_F32, "store_bf16": _lib.EPI_NONE, "accum_bf16": _lib.EPI_ACCUM}[epi]
    if simt and epi != "store_f32":
        pytest.skip("the exact-fp32 kernel writes f32")
    if simt:
        a, b = a.float(), b.float()
    ops.gemm(a, b, c, a_mn_major=True, b_mn_major=True, epilogue=code, valid_k=vk, simt=simt)
    ref = torch.zeros(B, rows, N, device=cuda, dtype=torch.float64)
    for e in range(B):
        kv = int(vk[e])
        ref[e] = a[e, :kv].double().T @ b[e, :kv].double()
    if epi == "accum_bf16":
        ref = ref + c0.double()
    got = c.double()
    assert torch.isfinite(got).all()
    tol = 1e-4 if dt == torch.float32 else 2e-2
    assert ((got - ref).abs() <= tol * ref.abs() + tol * ref.abs().max()).all()
    # valid_rows: rows of tiles at or past valid are not written
    rows_a = torch.randn(2, 384, 128, device=cuda, generator=g).bfloat16()
    w = torch.randn(2, 256, 128, device=cuda, generator=g).bfloat16()
    out = torch.full((2, 384, 256), 7.0, device=cuda, dtype=torch.float32)
    vr = torch.tensor([100, 0], device=cuda, dtype=torch.int32)
    if simt:
        rows_a, w = rows_a.float(), w.float()
    ops.gemm(rows_a, w, out, epilogue=_lib.EPI_STORE_F32, valid_rows=vr, simt=simt)
    full = torch.bmm(rows_a.double(), w.double().transpose(1, 2))
    assert torch.allclose(out[0, :100].double(), full[0, :100], rtol=1e-3, atol=1e-3)
    assert bool((out[1] == 7.0).all())  # expert with no routed rows: untouched


@pytest.mark.parametrize("T,M,E,k,renorm,cf,dtype", [(2048, 512, 64, 2, True, 1.0, "bf16"),
                                                     (1024, 256, 32, 1, True, 0.8, "bf16"),
                                                     (1000, 256, 16, 2, False, 1.0, "bf16"),
                                                     (4096, 512, 8, 2, True, 0.7, "bf16"),
                                                     (1024, 256, 6, 1, True, 1.0, "bf16"),
                                                     (2048, 256, 40, 4, False, 1.2, "bf16"),
                                                     (1024, 256, 64, 8, True, 1.0, "bf16"),
                                                     (512, 128, 16, 2, True, 1.0, "f32"),
                                                     (512, 128, 16, 1, True, 1.0, "f32")])
def test_combine_bwd_gate_route_matches_oracle(cuda, T, M, E, k, renorm, cf, dtype):
    """The layer's backward route (mpm_combine_bwd_gate -> mpm_gate_backward_gemms -> mpm_gate_gather):
    g_o bit-identical to mpm_combine_bwd's, dprob / dlogits / dWg / dx against the oracle's gate
    gradient (sparse gate term for top-k renormalisation, dense otherwise; drops on)."""
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator().manual_seed(T + M + k)
    x = torch.randn(T, M, generator=g).to(dt)
    wg = torch.randn(E, M, generator=g) / M ** 0.5
    C = O.capacity(T, k, E, cf)
    r = ops.compute_routing(x.to(cuda), wg.to(cuda), k, C, renorm)
    t_o = torch.randn(E * C, M, generator=g).to(dt).to(cuda)
    dy = torch.randn(T, M, generator=g).to(dt).to(cuda)
    g_i = torch.randn(E * C, M, generator=g).to(dt).to(cuda)
    ws = ops.gate_workspace(T, M, E, cuda)
    dl = torch.empty(T, E, device=cuda)
    dprob = torch.empty(T, k, device=cuda)
    g_o = torch.full((E * C, M), float("nan"), device=cuda, dtype=dt)
    ops.combine_bwd_gate(dy, t_o, r, 2, g_o, dl, ws, renorm, dprob=dprob)
    dwg = torch.empty(E, M, device=cuda)
    dx = torch.full((T, M), float("nan"), device=cuda, dtype=dt)
    ops.gate_backward_gemms(x.to(cuda), wg.to(cuda), dl, k, renorm, dwg, dx, ws)
    ops.gate_gather(r, g_i, wg.to(cuda), 2, dl, renorm, dx, ws)
    g_o_ref = torch.full_like(g_o, float("nan"))
    dprob_ref = ops.combine_bwd(dy, t_o, r, 2, g_o_ref)
    torch.cuda.synchronize()
    assert torch.equal(g_o, g_o_ref)
    assert torch.equal(dprob, dprob_ref)  # same fixed-order dot products
    idx, w, slot = r.idx.cpu().numpy(), r.weights.cpu().numpy(), r.slot.cpu().numpy()
    dl_ref = O.gate_grad(r.logits.cpu().numpy(), idx, w, dprob.cpu().numpy(), renorm)
    _close(dl.cpu().numpy(), dl_ref, 1e-5, 1e-6)
    _close(dwg.cpu().numpy(), dl_ref.T @ x.double().numpy(), 1e-4, 1e-5)
    dx_ref = dl_ref @ wg.double().numpy()
    gi = g_i.double().cpu().numpy()
    for j in range(k):
        keep = slot[:, j] >= 0
        C_ = C
        rows = idx[keep, j] * C_ + slot[keep, j]  # n_chunks only splits slots; rows stay e*C + s
        dx_ref[keep] += gi[rows]
    tol = 1e-2 if dtype == "bf16" else 1e-5
    _close(dx.double().cpu().numpy(), dx_ref, tol, tol)
