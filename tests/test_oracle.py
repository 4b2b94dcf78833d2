"""Pin the CPU oracle before trusting it.

The reference holds no MoE numerics, so the data-plane oracle is
checked against an independent restatement: a per-token torch-autograd
formula (no buffers, no all-to-all, no chunks) in float64.  Matching it shows
the oracle's slot layout, block-transposed all-to-all, chunking and
hand-written backward are all consistent with y[t] = sum_j w_j FFN_{e_j}(x_t).
"""

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O


def autograd_reference(xs, wg, w1s, w2s, dys, routing, renorm):
    N = len(xs)
    W1 = torch.tensor(np.concatenate(w1s), dtype=torch.float64, requires_grad=True)
    W2 = torch.tensor(np.concatenate(w2s), dtype=torch.float64, requires_grad=True)
    Wg = torch.tensor(wg, dtype=torch.float64, requires_grad=True)
    X = [torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in xs]
    loss = 0
    ys = []
    for r in range(N):
        ro = routing[r]
        logits = X[r] @ Wg.T
        idx = torch.tensor(ro.idx, dtype=torch.long)
        chosen = torch.gather(logits, 1, idx)
        if idx.shape[1] > 1 and renorm:
            w = torch.softmax(chosen, dim=1)
        else:
            w = torch.gather(torch.softmax(logits, dim=1), 1, idx)
        keep = torch.tensor(ro.slot >= 0, dtype=torch.float64)
        y = torch.zeros_like(X[r])
        for j in range(idx.shape[1]):
            h = torch.relu(torch.einsum("thm,tm->th", W1[idx[:, j]], X[r]))
            o = torch.einsum("tmh,th->tm", W2[idx[:, j]], h)
            y = y + (keep[:, j] * w[:, j])[:, None] * o
        ys.append(y)
        loss = loss + (y * torch.tensor(dys[r], dtype=torch.float64)).sum()
    loss.backward()
    E_loc = w1s[0].shape[0]
    return ([y.detach().numpy() for y in ys], [x.grad.numpy() for x in X], Wg.grad.numpy(),
            [W1.grad[r * E_loc:(r + 1) * E_loc].numpy() for r in range(N)],
            [W2.grad[r * E_loc:(r + 1) * E_loc].numpy() for r in range(N)])


@pytest.mark.parametrize("N,E,k,T,n,cf,renorm", [
    (1, 4, 1, 64, 2, 1.0, True),
    (1, 8, 2, 50, 3, 1.0, True),
    (2, 4, 2, 40, 2, 1.25, True),
    (2, 8, 1, 33, 1, 0.5, True),     # heavy drops
    (4, 8, 3, 24, 4, 1.0, False),    # raw top-k probabilities
])
def test_oracle_matches_autograd(N, E, k, T, n, cf, renorm):
    rng = np.random.default_rng(N * 100 + E + k)
    M, H = 12, 20
    xs = [rng.standard_normal((T, M)) for _ in range(N)]
    wg = rng.standard_normal((E, M))
    w1s = [rng.standard_normal((E // N, H, M)) * 0.3 for _ in range(N)]
    w2s = [rng.standard_normal((E // N, M, H)) * 0.3 for _ in range(N)]
    dys = [rng.standard_normal((T, M)) for _ in range(N)]
    res = O.moe_layer(xs, wg, w1s, w2s, k=k, capacity_factor=cf, n_chunks=n, renorm=renorm, dys=dys)
    y, dx, dwg, dw1, dw2 = autograd_reference(xs, wg, w1s, w2s, dys, res.routing, renorm)
    # the oracle derives routing weights from fp32 logits (the GPU's logits
    # dtype); autograd differentiates fp64 logits -> agreement to ~1e-7
    tol = dict(rtol=1e-6, atol=1e-6)
    for r in range(N):
        np.testing.assert_allclose(res.y[r], y[r], **tol)
        np.testing.assert_allclose(res.dx[r], dx[r], **tol)
        np.testing.assert_allclose(res.dw1[r], dw1[r], **tol)
        np.testing.assert_allclose(res.dw2[r], dw2[r], **tol)
    np.testing.assert_allclose(res.dwg, dwg, **tol)


def test_results_do_not_depend_on_chunking():
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal((96, 8)) for _ in range(2)]
    wg = rng.standard_normal((4, 8))
    w1s = [rng.standard_normal((2, 16, 8)) for _ in range(2)]
    w2s = [rng.standard_normal((2, 8, 16)) for _ in range(2)]
    dys = [rng.standard_normal((96, 8)) for _ in range(2)]
    base = O.moe_layer(xs, wg, w1s, w2s, k=2, capacity_factor=1.0, n_chunks=1, dys=dys)
    for n in (2, 5, 48):
        other = O.moe_layer(xs, wg, w1s, w2s, k=2, capacity_factor=1.0, n_chunks=n, dys=dys)
        for r in range(2):
            np.testing.assert_allclose(other.y[r], base.y[r], rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(other.dw1[r], base.dw1[r], rtol=1e-10, atol=1e-10)


def test_assign_slots_fast_equals_reference_loop():
    rng = np.random.default_rng(3)
    for T, E, k, C in [(100, 4, 1, 30), (257, 16, 2, 20), (64, 8, 4, 100), (1, 2, 1, 1), (50, 5, 2, 0)]:
        idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
        a = O.assign_slots(idx, E, C)
        b = O.assign_slots_fast(idx, E, C)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])


def test_route_tie_break_and_weights():
    logits = np.array([[1.0, 3.0, 3.0, 0.5], [2.0, 2.0, 2.0, 2.0]], dtype=np.float32)
    idx, w = O.route(logits, 2, True)
    np.testing.assert_array_equal(idx, [[1, 2], [0, 1]])   # equal logits -> lower index first
    np.testing.assert_allclose(w, [[0.5, 0.5], [0.5, 0.5]])
    idx1, w1 = O.route(logits, 1, True)
    np.testing.assert_array_equal(idx1[:, 0], [1, 0])
    np.testing.assert_allclose(w1[1, 0], 0.25)


def test_capacity_and_partitions():
    assert O.capacity(16384, 2, 64, 1.0) == 512      # cfg2
    assert O.capacity(8192, 1, 128, 1.25) == 80       # cfg5
    assert O.capacity(2048, 1, 4, 1.0) == 512         # cfg1
    assert O.partition_sizes(512, 4) == [128] * 4
    assert O.partition_sizes(10, 3) == [4, 3, 3]      # reference core.py:102-105
    assert O.chunk_starts(10, 3) == [0, 4, 7]


def test_oracle_matches_frozen_data_plane_vectors():
    """The oracle's outputs on seeded inputs equal tests/golden/data_plane.json (generated by
    tests/golden/gen_data_plane.py): routing exactly, float outputs by fingerprint (fp64 oracle,
    rtol 1e-9) — pins the data-plane semantics the reference leaves unpinned."""
    import json
    from pathlib import Path

    import numpy as np

    sys_path_root = Path(__file__).resolve().parent / "golden"
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen_data_plane", sys_path_root / "gen_data_plane.py")
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    frozen = json.loads((sys_path_root / "data_plane.json").read_text())
    for name, c in gen.CASES.items():
        got = gen.summarize(c)
        want = frozen[name]
        for r in range(c["N"]):
            for key in ("idx", "slot", "kept"):
                assert got["routing"][r][key] == want["routing"][r][key], (name, r, key)
            for key in ("y", "dx", "dw1", "dw2"):
                g_, w_ = got[key][r], want[key][r]
                for f in ("sum", "abs_sum", "l2"):
                    assert abs(g_[f] - w_[f]) <= 1e-9 * max(abs(w_[f]), 1.0), (name, r, key, f)
                np.testing.assert_allclose(g_["samples"], w_["samples"], rtol=1e-9, atol=1e-12)
        assert abs(got["dwg"]["l2"] - want["dwg"]["l2"]) <= 1e-9 * want["dwg"]["l2"]


def test_mask_override_layout_matches_computed_relu():
    """mask_override pins the ReLU per (local expert, source, slot): feeding the oracle the mask its
    own forward computes (gathered from a one-chunk run) reproduces the unpinned result for any
    chunking."""
    rng = np.random.default_rng(3)
    N, T, M, H, E, k = 2, 40, 8, 16, 4, 2
    xs = [rng.standard_normal((T, M)) for _ in range(N)]
    dys = [rng.standard_normal((T, M)) for _ in range(N)]
    wg = rng.standard_normal((E, M))
    w1s = [rng.standard_normal((E // N, H, M)) for _ in range(N)]
    w2s = [rng.standard_normal((E // N, M, H)) for _ in range(N)]
    base1 = O.moe_layer(xs, wg, w1s, w2s, k=k, capacity_factor=1.0, n_chunks=1, dys=dys)
    C = base1.extras["capacity"]
    masks = []
    for d in range(N):  # the one-chunk expert-side rows: [E_loc][src][slot]
        rows = []
        for el in range(E // N):
            e = d * (E // N) + el
            t_di = []
            for s in range(N):
                buf = np.zeros((C, M))
                ro = base1.routing[s]
                for j in range(k):
                    keep = ro.slot[:, j] >= 0
                    sel = keep & (ro.idx[:, j] == e)
                    buf[ro.slot[sel, j]] = xs[s][sel]
                t_di.append(buf)
            rows.append(np.concatenate(t_di) @ w1s[d][el].T > 0)
        masks.append(np.stack(rows))
    for n in (1, 3):
        ref = O.moe_layer(xs, wg, w1s, w2s, k=k, capacity_factor=1.0, n_chunks=n, dys=dys)
        pin = O.moe_layer(xs, wg, w1s, w2s, k=k, capacity_factor=1.0, n_chunks=n, dys=dys, mask_override=masks)
        for a, b in zip(ref.y + ref.dx + ref.dw1 + ref.dw2, pin.y + pin.dx + pin.dw1 + pin.dw2):
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
