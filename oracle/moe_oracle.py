"""CPU oracle for the MPipeMoE data plane — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker (never as the thing
measured or shipped).  The product path (paper_2506_22175_b200) never
imports it.

PARITY STATUS: the reference (`/root/reference`, package `moepipesim`) has
NO numerical MoE implementation (SPEC.md:14 puts "actual CUDA/NCCL
execution, PyTorch integration ... top-k routing dynamics" out of scope; the
paper's pmoe library is not vendored).  The data-plane
semantics below are therefore restated from the paper's prose and pinned
here; they are *unpinned by the reference* (SURVEY.md §8c).  What is pinned
against the reference is the control plane (chunk split, schedule, pools,
memory/cost models, Alg. 1 — see tests/golden/).  The oracle is
cross-checked against an independent torch-autograd restatement
(tests/test_oracle.py).

Semantics (one MoE layer, N ranks simulated in one process):
  * EP dataflow T_I -> T_DI -> T_M -> T_DO -> T_O:
    gate, dispatch all-to-all, expert FFN (two linear layers + activation),
    combine all-to-all, weighted combine.
  * Gate: logits = x . W_g^T in fp32/fp64 (E*M gate parameters, PAPER.md:180
    Eq. 1); top-k on the logits with the lowest expert index winning exact
    ties ("top-k algorithm"); weights = softmax probability of
    the chosen expert for k == 1, softmax over the k chosen logits
    (= renormalised top-k probabilities) for k > 1.
  * Capacity C = ceil(capacity_factor * T * k / E) slots per (source rank,
    expert); slots are granted in priority order (k-rank, token index);
    assignments beyond C are dropped and contribute 0 to the output.
  * Expert FFN: T_M = relu(T_DI . W1^T), T_DO = T_M . W2^T.  ReLU because the
    paper stores only the post-activation tensor and applies the activation
    in place ("in-place operations can be applied here"), which
    requires an activation whose derivative is a function of its output.
  * Pipelining: the capacity C is split into n chunks with the reference's
    balanced rule (core.py:102-105); chunk i carries slot range i of every
    (source rank, expert) block, i.e. the batch is split along the token
    dimension and each chunk is one full all-to-all.
    Weight gradients accumulate over chunks in chunk order.
  * Data parallelism for the gate: dW_g is summed over ranks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def capacity(tokens: int, k: int, num_experts: int, capacity_factor: float) -> int:
    """Slots per (source rank, expert): ceil(cf * T * k / E)."""
    return int(np.ceil(capacity_factor * tokens * k / num_experts - 1e-9))


def partition_sizes(total: int, n: int) -> list[int]:
    """Balanced split (reference core.py:102-105): first `total mod n` parts +1."""
    if n < 1 or n > max(total, 1):
        raise ValueError(f"cannot split {total} into {n} parts")
    base, extra = divmod(total, n)
    return [base + 1] * extra + [base] * (n - extra)


def chunk_starts(total: int, n: int) -> list[int]:
    sizes = partition_sizes(total, n)
    return [int(sum(sizes[:i])) for i in range(n)]


def gate_logits(x: np.ndarray, wg: np.ndarray) -> np.ndarray:
    """logits[T, E] = x . W_g^T, accumulated in float64."""
    return (x.astype(np.float64) @ wg.astype(np.float64).T)


def route(logits: np.ndarray, k: int, renorm: bool = True) -> tuple[np.ndarray, np.ndarray]:
    """Top-k expert indices (lowest index wins ties) and routing weights.

    Indices are decided on the fp32 logits exactly as given, so identical
    logits give bit-identical indices on every implementation.
    """
    lg = np.asarray(logits, dtype=np.float32)
    T, E = lg.shape
    # stable descending order on (-value, index): ties -> lower index first
    order = np.lexsort((np.broadcast_to(np.arange(E), (T, E)), -lg), axis=1)
    idx = order[:, :k].astype(np.int32)
    chosen = np.take_along_axis(lg, idx, axis=1).astype(np.float64)
    mx = chosen[:, :1]
    if k > 1 and renorm:
        ex = np.exp(chosen - mx)
        w = ex / ex.sum(axis=1, keepdims=True)
    else:
        den = np.exp(lg.astype(np.float64) - mx).sum(axis=1, keepdims=True)
        w = np.exp(chosen - mx) / den
    return idx, w


def assign_slots(idx: np.ndarray, num_experts: int, cap: int) -> tuple[np.ndarray, np.ndarray]:
    """Capacity-bounded slots, priority (k-rank, token index); -1 = dropped.

    Returns (slot[T, k] int32, kept[E] int32).
    """
    T, k = idx.shape
    slot = np.full((T, k), -1, dtype=np.int32)
    fill = np.zeros(num_experts, dtype=np.int64)
    for j in range(k):
        for t in range(T):
            e = int(idx[t, j])
            if fill[e] < cap:
                slot[t, j] = fill[e]
            fill[e] += 1
    kept = np.minimum(fill, cap).astype(np.int32)
    return slot, kept


def assign_slots_fast(idx: np.ndarray, num_experts: int, cap: int) -> tuple[np.ndarray, np.ndarray]:
    """Vectorised assign_slots (same result; used at larger sizes)."""
    T, k = idx.shape
    flat = idx.T.reshape(-1).astype(np.int64)          # priority order (j, t)
    order = np.argsort(flat, kind="stable")
    sorted_e = flat[order]
    starts = np.searchsorted(sorted_e, np.arange(num_experts))
    rank = np.empty_like(flat)
    rank[order] = np.arange(flat.size) - starts[sorted_e]
    slot = np.where(rank < cap, rank, -1).astype(np.int32).reshape(k, T).T.copy()
    counts = np.bincount(flat, minlength=num_experts)
    return slot, np.minimum(counts, cap).astype(np.int32)


def relu(a):
    return np.maximum(a, 0)


@dataclass
class RankRouting:
    logits: np.ndarray
    idx: np.ndarray
    w: np.ndarray
    slot: np.ndarray
    kept: np.ndarray


@dataclass
class LayerResult:
    y: list[np.ndarray]
    routing: list[RankRouting]
    dx: list[np.ndarray] | None = None
    dwg: np.ndarray | None = None
    dw1: list[np.ndarray] | None = None
    dw2: list[np.ndarray] | None = None
    dprob: list[np.ndarray] | None = None
    extras: dict = field(default_factory=dict)


def moe_layer(xs, wg, w1s, w2s, *, k: int, capacity_factor: float, n_chunks: int = 1,
              renorm: bool = True, dys=None, logits_override=None, mask_override=None,
              dtype=np.float64) -> LayerResult:
    """Forward (+ backward when dys is given) of one MoE layer over N ranks.

    xs[r]  : [T, M] tokens of rank r          (data-parallel)
    wg     : [E, M] gate weight (replicated)
    w1s[r] : [E_loc, H, M] fc1 weights of rank r's local experts
    w2s[r] : [E_loc, M, H] fc2 weights
    dys[r] : [T, M] upstream gradient of rank r's output
    logits_override[r]: use these fp32 logits instead of computing them
    (pins routing at the logits boundary, SURVEY.md §7 hard part 1).
    mask_override[d]: bool [E_loc, N*C, H] (viewed as [E_loc, N, C, H]),
    rank d's ReLU mask per (local expert, source rank, slot) — the layout of
    a one-chunk step's expert-side rows: T_M = where(mask, pre, 0) and the
    backward's ReLU' = mask.  Pins the activation at its kink the way the
    logits pin routing: a pre-activation within rounding of 0 may land on
    either side in bf16-in/fp32-accumulate vs the oracle's arithmetic, and
    such a flip moves that row's weight gradient by O(1).
    """
    N = len(xs)
    T, M = xs[0].shape
    E = wg.shape[0]
    E_loc = E // N
    H = w1s[0].shape[1]
    C = capacity(T, k, E, capacity_factor)
    sizes = partition_sizes(C, n_chunks) if C > 0 else [0] * n_chunks
    starts = chunk_starts(C, n_chunks) if C > 0 else [0] * n_chunks
    f = lambda a: np.asarray(a, dtype=dtype)

    routing = []
    send = []  # per rank: [E, C, M] (expert, slot) rows, zero where unused
    for r in range(N):
        lg = logits_override[r] if logits_override is not None else gate_logits(xs[r], wg).astype(np.float32)
        idx, w = route(lg, k, renorm)
        slot, kept = assign_slots_fast(idx, E, C)
        buf = np.zeros((E, C, M), dtype=dtype)
        tt, jj = np.nonzero(slot >= 0)
        buf[idx[tt, jj], slot[tt, jj]] = f(xs[r])[tt]
        routing.append(RankRouting(np.asarray(lg, np.float32), idx, w, slot, kept))
        send.append(buf)

    # expert side, chunk by chunk: rows of expert (d, el) ordered (src, slot)
    t_o = [np.zeros((E, C, M), dtype=dtype) for _ in range(N)]
    cache = []  # per chunk per dest rank: (t_di, t_m)
    for i in range(n_chunks):
        lo, hi = starts[i], starts[i] + sizes[i]
        per_rank = []
        for d in range(N):
            experts = range(d * E_loc, (d + 1) * E_loc)
            t_di = np.stack([np.concatenate([send[s][e, lo:hi] for s in range(N)]) for e in experts])
            pre = t_di @ np.swapaxes(f(w1s[d]), 1, 2)
            if mask_override is not None:
                mk = np.asarray(mask_override[d], dtype=bool)
                mk = mk.reshape(E_loc, N, mk.shape[1] // N, mk.shape[2])
                act = mk[:, :, lo:hi, :].reshape(E_loc, N * (hi - lo), mk.shape[3])
                t_m = np.where(act, pre, 0).astype(dtype)
            else:
                act = pre > 0
                t_m = relu(pre)
            t_do = t_m @ np.swapaxes(f(w2s[d]), 1, 2)
            for el, e in enumerate(experts):
                for s in range(N):
                    t_o[s][e, lo:hi] = t_do[el, s * (hi - lo):(s + 1) * (hi - lo)]
            per_rank.append((t_di, t_m, act))
        cache.append(per_rank)

    ys = []
    for r in range(N):
        ro = routing[r]
        y = np.zeros((T, M), dtype=dtype)
        for j in range(k):
            keep = ro.slot[:, j] >= 0
            rows = t_o[r][ro.idx[keep, j], ro.slot[keep, j]]
            y[keep] += ro.w[keep, j:j + 1].astype(dtype) * rows
        ys.append(y)
    res = LayerResult(y=ys, routing=routing)
    if dys is None:
        return res

    # ---------------- backward
    g_o, dprobs = [], []
    for r in range(N):
        ro = routing[r]
        dy = f(dys[r])
        buf = np.zeros((E, C, M), dtype=dtype)
        dp = np.zeros((T, k), dtype=dtype)
        for j in range(k):
            keep = np.nonzero(ro.slot[:, j] >= 0)[0]
            e, s = ro.idx[keep, j], ro.slot[keep, j]
            dp[keep, j] = np.einsum("tm,tm->t", dy[keep], t_o[r][e, s])
            buf[e, s] = ro.w[keep, j:j + 1].astype(dtype) * dy[keep]
        g_o.append(buf)
        dprobs.append(dp)

    dw1 = [np.zeros((E_loc, H, M), dtype=dtype) for _ in range(N)]
    dw2 = [np.zeros((E_loc, M, H), dtype=dtype) for _ in range(N)]
    g_i = [np.zeros((E, C, M), dtype=dtype) for _ in range(N)]
    for i in range(n_chunks):
        lo, hi = starts[i], starts[i] + sizes[i]
        for d in range(N):
            experts = range(d * E_loc, (d + 1) * E_loc)
            t_di, t_m, act = cache[i][d]
            g_do = np.stack([np.concatenate([g_o[s][e, lo:hi] for s in range(N)]) for e in experts])
            d_tm = g_do @ f(w2s[d])                       # [E_loc, R, H]
            d_h = d_tm * act
            dw2[d] += np.swapaxes(g_do, 1, 2) @ t_m       # [E_loc, M, H]
            g_di = d_h @ f(w1s[d])                        # [E_loc, R, M]
            dw1[d] += np.swapaxes(d_h, 1, 2) @ t_di       # [E_loc, H, M]
            for el, e in enumerate(experts):
                for s in range(N):
                    g_i[s][e, lo:hi] = g_di[el, s * (hi - lo):(s + 1) * (hi - lo)]

    dxs = []
    dwg = np.zeros((E, M), dtype=dtype)
    dlogits_all = []
    for r in range(N):
        ro = routing[r]
        dl = gate_grad(ro.logits, ro.idx, ro.w, dprobs[r], renorm).astype(dtype)
        dx = dl @ f(wg)
        for j in range(k):
            keep = ro.slot[:, j] >= 0
            dx[keep] += g_i[r][ro.idx[keep, j], ro.slot[keep, j]]
        dxs.append(dx)
        dwg += dl.T @ f(xs[r])
        dlogits_all.append(dl)
    res.dx, res.dwg, res.dw1, res.dw2, res.dprob = dxs, dwg, dw1, dw2, dprobs
    res.extras["dlogits"] = dlogits_all
    res.extras["capacity"] = C
    return res


def gate_grad(logits, idx, w, dprob, renorm: bool = True) -> np.ndarray:
    """d loss / d logits through the routing weights (softmax Jacobian)."""
    T, E = logits.shape
    k = idx.shape[1]
    w = w.astype(np.float64)
    dp = dprob.astype(np.float64)
    s = (w * dp).sum(axis=1, keepdims=True)
    out = np.zeros((T, E), dtype=np.float64)
    rows = np.arange(T)[:, None]
    if k > 1 and renorm:
        np.put_along_axis(out, idx.astype(np.int64), w * (dp - s), axis=1)
        return out
    lg = logits.astype(np.float64)
    p = np.exp(lg - lg.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    out = -p * s
    np.add.at(out, (np.broadcast_to(rows, idx.shape), idx.astype(np.int64)), w * dp)
    return out
