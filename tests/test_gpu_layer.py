"""End-to-end parity of MoELayer (forward + backward) against the CPU oracle.

Routing is pinned at the logits boundary: the oracle is fed the layer's own
fp32 logits, so indices / slots / drops must match bit for bit, and the
outputs and every gradient must match within the north-star tolerances
(fp32: rtol 1e-5; bf16: rtol 2e-2 vs the fp32/fp64 oracle).
"""

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from paper_2506_22175_b200.layer import MoELayer

pytestmark = pytest.mark.gpu


def _close(got, ref, rtol, atol_scale):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    atol = atol_scale * max(np.abs(ref).max(), 1e-30)
    viol = np.abs(got - ref) - (rtol * np.abs(ref) + atol)
    assert viol.max() <= 0, f"max violation {viol.max():.3e} (rtol {rtol}, atol {atol:.3e})"


def gpu_mask(arena) -> np.ndarray | None:
    """The arena's 1-bit ReLU mask as bool [E_loc, N*C, H] (expert-side all-chunk layout), or None
    (fp32 layers keep no mask; reuse arenas keep only ring slots)."""
    mf = arena.mask_full
    if mf is None:
        return None
    g = arena.g
    words = mf.view(g.e_loc, g.N * g.C, arena.mask_w)[:, :, : g.H // 32].contiguous().cpu().numpy()
    return np.unpackbits(words.view(np.uint8), axis=-1, bitorder="little").astype(bool)


def capture_mask(layer, x) -> np.ndarray | None:
    """The GPU's ReLU mask for x: a no-grad n=1 forward (fc1 rows do not depend on the chunking, so
    every n and strategy computes these bits; tests/test_gpu_layer.py asserts y/dx bit-identical)."""
    if layer.w1.dtype == torch.float32:
        return None
    with torch.no_grad():
        layer(x, n=1)
    return gpu_mask(layer.last_arena)


def run_layer(layer, x, dy, n, strategy=None):
    mask = capture_mask(layer, x)
    x = x.clone().requires_grad_(True)
    y = layer(x, n=n, strategy=strategy)
    y.backward(dy)
    step = layer.last_arena
    out = {
        "y": y.detach().float().cpu().numpy(),
        "dx": x.grad.float().cpu().numpy(),
        "dwg": layer.gate_weight.grad.float().cpu().numpy(),
        "dw1": layer.w1.grad.float().cpu().numpy(),
        "dw2": layer.w2.grad.float().cpu().numpy(),
        "logits": step.logits.cpu().numpy(),
        "idx": step.idx.cpu().numpy(),
        "slot": step.slot.cpu().numpy(),
        "kept": step.kept.cpu().numpy(),
        "mask": mask,
    }
    for p in layer.parameters():
        p.grad = None
    return out


def oracle_for(layer, x, dy, n, out, dtype=np.float64):
    """The oracle on the layer's inputs, with routing pinned at the GPU's fp32 logits and the ReLU
    pinned at the GPU's 1-bit mask (oracle/moe_oracle.py moe_layer)."""
    res = O.moe_layer([x.float().cpu().numpy()], layer.gate_weight.detach().cpu().numpy(),
                      [layer.w1.detach().float().cpu().numpy()], [layer.w2.detach().float().cpu().numpy()],
                      k=layer.top_k, capacity_factor=layer.capacity_factor, n_chunks=n,
                      renorm=layer.renorm, dys=[dy.float().cpu().numpy()], logits_override=[out["logits"]],
                      mask_override=None if out["mask"] is None else [out["mask"]], dtype=dtype)
    return res


def check(out, res, rtol, atol):
    """Routing bit-exact; y, dx, dWg, dW1, dW2 elementwise within rtol (+ atol x max|ref|)."""
    np.testing.assert_array_equal(out["idx"], res.routing[0].idx)
    np.testing.assert_array_equal(out["slot"], res.routing[0].slot)
    np.testing.assert_array_equal(out["kept"], res.routing[0].kept)
    for key, ref in (("y", res.y[0]), ("dx", res.dx[0]), ("dwg", res.dwg), ("dw1", res.dw1[0]),
                     ("dw2", res.dw2[0])):
        try:
            _close(out[key], ref, rtol, atol)
        except AssertionError as e:
            raise AssertionError(f"{key}: {e}") from None


def make(cuda, M, H, E, k, T, dtype, cf=1.0, seed=0, **kw):
    layer = MoELayer(M, H, E, top_k=k, capacity_factor=cf, pipeline=False, dtype=dtype, device=cuda, seed=seed, **kw)
    layer.record_times = True
    g = torch.Generator().manual_seed(1000 + seed)
    x = torch.randn(T, M, generator=g).to(dtype).to(cuda)
    dy = torch.randn(T, M, generator=g).to(dtype).to(cuda)
    return layer, x, dy


def test_cfg1_fp32_parity(cuda):
    """BASELINE.json configs[0]: 4 experts top-1, M=256, H=1024, 2048 tokens, n=2, fp32."""
    layer, x, dy = make(cuda, 256, 1024, 4, 1, 2048, torch.float32)
    out = run_layer(layer, x, dy, n=2)
    check(out, oracle_for(layer, x, dy, 2, out), 1e-5, 1e-5)


def test_fp32_uneven_chunks_two_lanes_parity(cuda):
    """fp32 (exact FMA kernels) with n=3 uneven chunks and no reuse: chunks 0/2 and 1 run on the
    two compute lanes; top-2 over 12 experts (padded gate operands), fp32 bars."""
    layer, x, dy = make(cuda, 128, 256, 12, 2, 1000, torch.float32, cf=1.1, seed=9)
    out = run_layer(layer, x, dy, n=3)
    assert layer.last_arena.lanes, "expected the second compute lane to be in use"
    check(out, oracle_for(layer, x, dy, 3, out), 1e-5, 1e-5)


def test_few_rows_per_expert_parity(cuda):
    """BASELINE configs[4]-like regime (many experts, top-1, cf 1.25): ~10 rows per expert, so the
    weight-gradient GEMMs have one k-block per tile and take the 8-warp epilogue."""
    layer, x, dy = make(cuda, 256, 1024, 64, 1, 512, torch.bfloat16, cf=1.25, seed=13)
    out = run_layer(layer, x, dy, n=1)
    check(out, oracle_for(layer, x, dy, 1, out), 2e-2, 2e-2)


def test_top8_routing_layer_parity(cuda):
    """k = 8 (the largest compiled top-k) over 16 experts, bf16, n=2."""
    layer, x, dy = make(cuda, 256, 512, 16, 8, 512, torch.bfloat16, cf=1.0, seed=11)
    out = run_layer(layer, x, dy, n=2)
    check(out, oracle_for(layer, x, dy, 2, out), 2e-2, 2e-2)


@pytest.mark.parametrize("n,strategy,acc", [(1, None, "param"), (2, "s4", "param"), (4, "s1", "param"),
                                            (3, "s2", "param"), (2, "s3", "param"), (4, "s4", "fp32"),
                                            (8, "s3", "param")])
def test_bf16_parity(cuda, n, strategy, acc):
    layer, x, dy = make(cuda, 512, 1024, 16, 2, 2048, torch.bfloat16, cf=1.25, seed=3, wgrad_accumulation=acc)
    out = run_layer(layer, x, dy, n=n, strategy=strategy)
    check(out, oracle_for(layer, x, dy, n, out), 2e-2, 2e-2)


def test_results_independent_of_granularity_and_strategy(cuda):
    """Chunking splits slots, not math: y and dx are bit-identical for every n and strategy."""
    layer, x, dy = make(cuda, 256, 512, 8, 2, 1024, torch.bfloat16, seed=5)
    base = run_layer(layer, x, dy, n=1)
    for n, strat in [(2, None), (4, "s4"), (4, "s3"), (8, "s1"), (2, "s2")]:
        out = run_layer(layer, x, dy, n=n, strategy=strat)
        np.testing.assert_array_equal(out["y"], base["y"])
        np.testing.assert_array_equal(out["dx"], base["dx"])
        _close(out["dw1"], base["dw1"], 1e-2, 1e-2)


def test_measured_trace_is_valid(cuda):
    from paper_2506_22175_b200.trace import replay_validate, to_jsonl
    layer, x, dy = make(cuda, 256, 1024, 8, 2, 4096, torch.bfloat16)
    for strat in (None, "s4", "s1"):
        run_layer(layer, x, dy, n=4, strategy=strat)
        fw, bw = layer.last_arena.traces()
        replay_validate(fw)
        replay_validate(bw)
        assert to_jsonl(fw).count("\n") == len(fw.dag.ops)


def test_cfg2_shape_full_size_properties(cuda):
    """cfg2 at N=1 (T=16K, E=64, k=2, M=1024, H=4096): finite, deterministic, routing self-consistent."""
    layer, x, dy = make(cuda, 1024, 4096, 64, 2, 16384, torch.bfloat16)
    a = run_layer(layer, x, dy, n=1)
    b = run_layer(layer, x, dy, n=1)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert np.isfinite(a[key]).all(), key
        np.testing.assert_array_equal(a[key], b[key])  # bitwise reproducible
    idx_ref, _ = O.route(a["logits"], 2, True)
    slot_ref, kept_ref = O.assign_slots_fast(idx_ref, 64, O.capacity(16384, 2, 64, 1.0))
    np.testing.assert_array_equal(a["idx"], idx_ref)
    np.testing.assert_array_equal(a["slot"], slot_ref)
    np.testing.assert_array_equal(a["kept"], kept_ref)


@pytest.mark.parametrize("M,H,E,k,T,n,strategy", [
    (1024, 4096, 64, 2, 16384, 1, None),     # BASELINE configs[1] shape at N=1
    (1024, 4096, 64, 2, 16384, 4, "s4"),     # same, pipelined with reuse
    (2048, 8192, 32, 1, 8192, 2, None),      # configs[2] at its smallest sweep point
    (4096, 16384, 64, 2, 8192, 2, "s3"),     # configs[3] dims (expert weights 17 GB bf16)
])
def test_full_size_exact_linearity(cuda, M, H, E, k, T, n, strategy):
    """Size-independent properties at the BASELINE dims, where the oracle is too slow:
    scaling W2 by 2 (exact in floating point) doubles y and dW1 bit for bit and leaves
    dW2 and the routing unchanged; every output is finite; assignment conserves tokens.
    Compared on the device (the cfg4-sized weight gradients are 8.6 G elements)."""
    layer, x, dy = make(cuda, M, H, E, k, T, torch.bfloat16)

    def step():
        xg = x.clone().requires_grad_(True)
        y = layer(xg, n=n, strategy=strategy)
        y.backward(dy)
        st = layer.last_arena
        out = {"y": y.detach(), "dx": xg.grad, "dwg": layer.gate_weight.grad, "dw1": layer.w1.grad,
               "dw2": layer.w2.grad, "idx": st.idx.clone(), "slot": st.slot.clone(), "kept": st.kept.clone(),
               "logits": st.logits.clone()}
        for p in layer.parameters():
            p.grad = None
        return out

    a = step()
    with torch.no_grad():
        layer.w2.mul_(2)
    b = step()
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert bool(torch.isfinite(a[key]).all()), key
    for key in ("idx", "slot", "kept", "logits"):
        assert torch.equal(a[key], b[key]), key
    assert torch.equal(b["y"], 2 * a["y"])
    assert torch.equal(b["dw1"], 2 * a["dw1"])
    assert torch.equal(b["dw2"], a["dw2"])
    C = O.capacity(T, k, E, 1.0)
    idx, slot, kept = a["idx"].cpu().numpy(), a["slot"].cpu().numpy(), a["kept"].cpu().numpy()
    assert (slot >= 0).sum() == kept.sum() and kept.max() <= C
    assert np.bincount(idx[slot >= 0], minlength=E).tolist() == kept.tolist()


def test_reuse_lowers_arena_bytes(cuda):
    """Memory reuse (ring slots + in-place bf16 wgrad accumulation) must shrink the step's
    device footprint below the no-reuse pipeline at the same n (Eq. 5)."""
    layer, x, dy = make(cuda, 512, 2048, 8, 2, 8192, torch.bfloat16)
    sizes = {}
    for strat in (None, "s4", "s3", "s1"):
        run_layer(layer, x, dy, n=4, strategy=strat)
        sizes[strat] = layer.last_arena.device_bytes
        layer.release_arenas()
    for strat in ("s4", "s3", "s1"):
        assert sizes[strat] < sizes[None], sizes


@pytest.mark.parametrize("T,M,H,E,k,cf,n,skew", [
    (1000, 256, 512, 48, 4, 0.5, 2, False),   # top-4, E % 32 != 0 (padded gate), T % 64 != 0 (exact gate bwd), drops
    (2048, 256, 512, 8, 2, 1.0, 2, False),    # E = 8 (padded tensor-core gate forward and backward)
    (1024, 128, 256, 6, 1, 1.25, 1, False),   # E = 6: E % 4 != 0
    (500, 96, 160, 8, 2, 1.0, 2, False),      # M % 64 != 0 (exact gate, ragged K tiles), H/32 = 5 mask words
    (777, 128, 256, 24, 3, 1.0, 3, False),    # odd top-k (k=3 on the KM=4 kernels), E=24, uneven chunks
    (77, 128, 256, 8, 1, 2.0, 1, False),      # tiny ragged batch, spare capacity (zero-filled slots)
    (4096, 256, 512, 16, 2, 1.0, 4, True),    # skewed gate: a quarter of the experts overloaded -> drops
])
def test_layer_edge_shapes(cuda, T, M, H, E, k, cf, n, skew):
    layer, x, dy = make(cuda, M, H, E, k, T, torch.bfloat16, cf=cf, seed=7)
    if skew:
        with torch.no_grad():
            layer.gate_weight[: E // 4] *= 4.0
    out = run_layer(layer, x, dy, n=n)
    res = oracle_for(layer, x, dy, n, out)
    check(out, res, 2e-2, 2e-2)
    C = O.capacity(T, k, E, cf)
    if skew:
        assert (out["slot"] < 0).any(), "the skewed gate should overflow some experts"
    assert out["kept"].max() <= C


def test_idle_arena_cache_is_bounded(cuda):
    """Dynamic batch sizes: one arena per token count, but at most max_cached_arenas stay cached."""
    layer = MoELayer(128, 256, 8, top_k=2, pipeline=1, dtype=torch.bfloat16, device=cuda, max_cached_arenas=2)
    for T in (256, 320, 384, 448, 512, 256):
        x = torch.randn(T, 128, device=cuda).bfloat16().requires_grad_(True)
        layer(x).sum().backward()
        idle = sum(len(v) for v in layer._arenas.values())
        assert idle <= 2, idle


def test_algorithm1_state_survives_state_dict(cuda):
    """Algorithm 1's learned ranges and the measured profile ride along in state_dict() and are
    reused after load_state_dict() (no re-search on a resumed job)."""
    layer = MoELayer(128, 256, 8, top_k=2, pipeline="adaptive", memory_reuse="auto", dtype=torch.bfloat16,
                     device=cuda, candidates=(1, 2))
    n1, strat1, _ = layer.plan(512)
    sd = layer.state_dict()
    fresh = MoELayer(128, 256, 8, top_k=2, pipeline="adaptive", memory_reuse="auto", dtype=torch.bfloat16,
                     device=cuda, candidates=(1, 2))
    fresh.load_state_dict(sd)
    n2, strat2, _ = fresh.plan(512)
    assert (n1, strat1.name) == (n2, strat2.name)
    assert fresh._controller.stats.searches == 0 and fresh._controller.stats.cache_hits == 1


# ---------------------------------------------------------------- BASELINE layer dims vs the oracle
@pytest.mark.parametrize("n,strategy,acc", [(1, None, "param"), (4, None, "param"), (4, "s4", "param"),
                                            (4, "s3", "fp32")])
def test_cfg2_dims_oracle_parity(cuda, n, strategy, acc):
    """BASELINE configs[1] layer dims at N=1 (M=1024, H=4096, all 64 experts local, top-2, bf16) at 4K
    tokens: the 64-way batched GEMMs of the headline shape against the fp32 oracle, elementwise."""
    layer, x, dy = make(cuda, 1024, 4096, 64, 2, 4096, torch.bfloat16, seed=21, wgrad_accumulation=acc)
    out = run_layer(layer, x, dy, n=n, strategy=strategy)
    check(out, oracle_for(layer, x, dy, n, out, dtype=np.float32), 2e-2, 2e-2)


def test_cfg3_dims_oracle_parity(cuda):
    """BASELINE configs[2] layer dims (M=2048, H=8192, E=32, top-1) at 2K tokens, n=2."""
    layer, x, dy = make(cuda, 2048, 8192, 32, 1, 2048, torch.bfloat16, seed=22)
    out = run_layer(layer, x, dy, n=2)
    check(out, oracle_for(layer, x, dy, 2, out, dtype=np.float32), 2e-2, 2e-2)


def test_cfg5_layer_oracle_parity(cuda):
    """BASELINE configs[4]'s MoE layer (M=1024, H=4096, 128 experts top-1, capacity factor 1.25) at
    8K tokens (8 sequences of 1024): ~80 capacity rows per expert, padded slots, drops."""
    layer, x, dy = make(cuda, 1024, 4096, 128, 1, 8192, torch.bfloat16, cf=1.25, seed=23)
    out = run_layer(layer, x, dy, n=1)
    check(out, oracle_for(layer, x, dy, 1, out, dtype=np.float32), 2e-2, 2e-2)


def test_routing_from_x_end_to_end(cuda):
    """Routing from the tokens, not from the layer's logits: the oracle computes fp64 logits from x
    and W_g and routes on them; indices must agree everywhere except where the k-th and (k+1)-th
    logits of a token are within the gate's fp32 rounding (|gap| <= 1e-5 * scale), and every such
    token is counted (a few at most)."""
    layer, x, dy = make(cuda, 1024, 4096, 64, 2, 16384, torch.bfloat16, seed=24)
    with torch.no_grad():
        layer(x, n=1)
    a = layer.last_arena
    lg_gpu = a.logits.cpu().numpy()
    idx_gpu = a.idx.cpu().numpy()
    lg_ref = O.gate_logits(x.float().cpu().numpy(), layer.gate_weight.detach().cpu().numpy())
    scale = np.abs(lg_ref).max()
    np.testing.assert_allclose(lg_gpu, lg_ref, rtol=0, atol=1e-5 * scale)  # fp32-accurate gate
    idx_ref, _ = O.route(lg_ref.astype(np.float32), 2, True)
    srt = -np.sort(-lg_ref, axis=1)
    near_tie = (srt[:, 0] - srt[:, 1] <= 1e-5 * scale) | (srt[:, 1] - srt[:, 2] <= 1e-5 * scale)
    differ = (np.sort(idx_gpu, 1) != np.sort(idx_ref, 1)).any(axis=1)
    assert not (differ & ~near_tie).any(), f"{(differ & ~near_tie).sum()} tokens routed differently"
    assert differ.sum() <= 8, differ.sum()


@pytest.mark.parametrize("n,strategy", [(1, None), (3, None), (2, "s4")])
def test_padding_skip_is_exact(cuda, n, strategy):
    """Skipping the capacity padding (row tiles / K blocks past each expert's routed tokens, N = 1)
    changes no bit: the skipped rows only ever contribute exact zeros.  Skewed gate, cf 1.25."""
    layer, x, dy = make(cuda, 256, 512, 16, 2, 4096, torch.bfloat16, cf=1.25, seed=31)
    with torch.no_grad():
        layer.gate_weight[:4] *= 3.0
    on = run_layer(layer, x, dy, n=n, strategy=strategy)
    assert layer.last_arena.skip_padding
    layer._skip_padding = False
    layer.release_arenas()
    off = run_layer(layer, x, dy, n=n, strategy=strategy)
    assert not layer.last_arena.skip_padding
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        np.testing.assert_array_equal(on[key], off[key], err_msg=key)
