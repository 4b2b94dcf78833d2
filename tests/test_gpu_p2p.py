"""The production N > 1 path: MoELayer over comm.PeerComm (IPC windows +
copy-engine chunk exchanges + stream-memory-op flags, csrc/p2p.cu) in real
separate processes, all sharing the one GPU of the box, against the N-rank
CPU oracle.  Routing bit-exact; outputs and gradients within the bf16 bars;
the all-reduced gate gradient bitwise identical on every rank.  Two steps
per run, so the second reuses the arena and catches stale-flag (a flag not
reset by its last waiter) or buffer-reuse hazards.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import moe_oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _close(got, ref, rtol, atol_scale):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    atol = atol_scale * max(np.abs(ref).max(), 1e-30)
    viol = np.abs(got - ref) > rtol * np.abs(ref) + atol
    assert not viol.any(), f"{viol.sum()} of {viol.size} outside tolerance"


def _free_port() -> int:
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _run(tmp_path, world, n, strategy, env_extra=None, port=None, **shape):
    """torchrun the worker; the rendezvous port is picked free at run time (the `port`
    arguments only keep the parametrized test ids stable)."""
    port = _free_port()
    out = tmp_path / "p2p.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "p2p_worker.py"),
           "--out", str(out), "--chunks", str(n), "--strategy", strategy]
    for k_, v in shape.items():
        cmd += [f"--{k_}", str(v)]
    env = dict(os.environ, **(env_extra or {}))
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return dict(np.load(out))


def _check(d, world, n, k=2, cf=1.25, steps=2, rtol=2e-2, dtype=np.float64):
    """Every rank, every step: routing bit-exact (pinned at the logits), outputs and gradients
    elementwise within rtol (+ rtol x max|ref|), the ReLU pinned at each rank's GPU mask."""
    for s_ in range(steps):
        xs = [d[f"r{r}_s{s_}_x"] for r in range(world)]
        dys = [d[f"r{r}_s{s_}_dy"] for r in range(world)]
        res = O.moe_layer(xs, d["r0_wg"], [d[f"r{r}_w1"] for r in range(world)],
                          [d[f"r{r}_w2"] for r in range(world)], k=k, capacity_factor=cf, n_chunks=n, dys=dys,
                          logits_override=[d[f"r{r}_s{s_}_logits"] for r in range(world)],
                          mask_override=[d[f"r{r}_s{s_}_mask"] for r in range(world)]
                          if f"r0_s{s_}_mask" in d else None, dtype=dtype)
        for r in range(world):
            p = f"r{r}_s{s_}_"
            np.testing.assert_array_equal(d[p + "idx"], res.routing[r].idx)
            np.testing.assert_array_equal(d[p + "slot"], res.routing[r].slot)
            _close(d[p + "y"], res.y[r], rtol, rtol)
            _close(d[p + "dx"], res.dx[r], rtol, rtol)
            _close(d[p + "dwg"], res.dwg, rtol, rtol)
            _close(d[p + "dw1"], res.dw1[r], rtol, rtol)
            _close(d[p + "dw2"], res.dw2[r], rtol, rtol)
            np.testing.assert_array_equal(d[p + "dwg"], d[f"r0_s{s_}_dwg"])  # fixed-order sum: same bits


@pytest.mark.parametrize("n,strategy", [(1, "none"), (2, "none"), (3, "s4"), (2, "s1"), (4, "s3")])
def test_two_process_peer_memory_layer(tmp_path, n, strategy):
    d = _run(tmp_path, 2, n, strategy, port=29611 + n)
    _check(d, 2, n)


def test_ragged_tokens_uneven_chunks_two_process(tmp_path):
    """T=300 tokens (not a multiple of anything), 3 uneven chunks, S2 (re-dispatch + host offload)."""
    d = _run(tmp_path, 2, 3, "s2", port=29701, T=300, E=8, M=128, H=256)
    _check(d, 2, 3)


def test_four_process_peer_memory_layer(tmp_path):
    d = _run(tmp_path, 4, 2, "s4", port=29631, E=8)
    _check(d, 4, 2)


def test_adaptive_granularity_and_auto_reuse_two_process(tmp_path):
    """pipeline="adaptive" + memory_reuse="auto" across 2 processes: Algorithm 1 times real peer-memory
    steps (max over ranks), the strategy comes from a profile whose w_comm is a timed peer-memory
    exchange; every rank must take the same (n, strategy) and the step must match the oracle."""
    d = _run(tmp_path, 2, "adaptive", "auto", port=29691)
    n = int(d["r0_n"])
    assert int(d["r1_n"]) == n and str(d["r0_strategy"]) == str(d["r1_strategy"])
    _check(d, 2, n)


def test_cfg1_fp32_two_process(tmp_path):
    """BASELINE configs[0] (4 experts top-1, M=256, H=1024, 2048 tokens, n=2, fp32) expert-parallel over
    2 processes: fp32 bars (rtol 1e-5) against the 2-rank oracle."""
    d = _run(tmp_path, 2, 2, "none", port=29651, T=2048, M=256, H=1024, E=4, k=1, dtype="f32")
    _check(d, 2, 2, k=1, rtol=1e-5)


@pytest.mark.parametrize("n,strategy", [(2, "none"), (2, "s4")])
def test_four_process_cfg2_dims(tmp_path, n, strategy):
    """BASELINE configs[1] layer dims expert-parallel over 4 processes: M=1024, H=4096, E=64 (16
    experts per rank), top-2, 2K tokens per rank, cf 1.0, against the 4-rank oracle (fp32)."""
    d = _run(tmp_path, 4, n, strategy, T=2048, M=1024, H=4096, E=64, k=2, cf=1.0)
    _check(d, 4, n, k=2, cf=1.0, dtype=np.float32)


@pytest.mark.parametrize("cf,n", [(2.0, 2), (0.5, 1), (1.25, 3)])
def test_compacted_expert_side_two_process(tmp_path, cf, n):
    """The compacted expert side (fused dispatch): every source's routed rows of an expert follow the
    lower sources' rows, the GEMMs stop at the routed total.  cf 2.0: half the slots are padding;
    cf 0.5: drops; n = 3 over 4 local experts: uneven expert groups (every chunk one slot part)."""
    d = _run(tmp_path, 2, n, "none", cf=cf)
    assert bool(d["r0_compact"]) and bool(d["r1_compact"])
    _check(d, 2, n, cf=cf)


@pytest.mark.parametrize("world", [2, 4])
def test_compacted_skewed_routing(tmp_path, world):
    """Skewed routing on the compacted expert side: the two biased experts overflow (drops) while the
    others' loads differ widely between sources, so the compacted offsets, totals and 64-row zero
    tails vary per (source, expert)."""
    d = _run(tmp_path, world, 2, "none", skew=3.0, E=8, cf=1.0)
    assert bool(d["r0_compact"])
    _check(d, world, 2, cf=1.0)


@pytest.mark.parametrize("strategy,cf,skew", [("s4", 2.0, 0.0), ("s3", 1.0, 3.0), ("s1", 1.25, 0.0)])
def test_compacted_ring_pulls_two_process(tmp_path, strategy, cf, skew):
    """Memory reuse on the compacted expert side: the receiver pulls each source's routed rows into the
    ring slot at the lower sources' prefix (mpm_compact_pull, counts riding on TI_READY), per chunk slot
    range — E = 4 over 2 ranks at n = 4 gives two slot parts per expert group — with recompute (S4 / S3)
    or host offload (S1) of the compacted rows."""
    d = _run(tmp_path, 2, 4, strategy, E=4, cf=cf, skew=skew)
    assert bool(d["r0_compact"])
    _check(d, 2, 4, cf=cf)


def test_compaction_leaves_outputs_bitwise(tmp_path):
    """Compacted vs capacity expert-side layout (MPM_COMPACT=0): every token's rows go through the
    same GEMMs in the same K order, so y and dx are bit-identical; the weight gradients sum the same
    rows in another order (and skip exact zeros), so they agree to rounding."""
    (tmp_path / "a").mkdir()
    (tmp_path / "b").mkdir()
    da = _run(tmp_path / "a", 2, 2, "none")
    db = _run(tmp_path / "b", 2, 2, "none", env_extra={"MPM_COMPACT": "0"})
    assert bool(da["r0_compact"]) and not bool(db["r0_compact"])
    for r in range(2):
        for s_ in range(2):
            p = f"r{r}_s{s_}_"
            np.testing.assert_array_equal(da[p + "y"], db[p + "y"])
            np.testing.assert_array_equal(da[p + "dx"], db[p + "dx"])
            _close(da[p + "dw1"], db[p + "dw1"], 2e-2, 2e-2)
            _close(da[p + "dw2"], db[p + "dw2"], 2e-2, 2e-2)


@pytest.mark.parametrize("n,strategy", [(2, "none"), (4, "s4")])
def test_eight_process_peer_memory_layer(tmp_path, n, strategy):
    """The north star's topology, N = 8 (one expert group per rank), as 8 processes sharing the GPU:
    E = 16 (2 experts per rank), top-2, every rank's chunks exchanged with 7 peers over the IPC
    windows, against the 8-rank oracle; the second step reuses the arena (flag reset / buffer reuse)."""
    d = _run(tmp_path, 8, n, strategy, T=256, M=128, H=256, E=16)
    _check(d, 8, n)


def test_bench_eight_ranks_self_check(tmp_path):
    """bench.py --gpus 8 under torchrun (8 ranks sharing this GPU through MPM_BENCH_BACKEND=gloo: a
    functional check of the N = 8 bench path, not a measurement): the JSON line reports 8 GPUs, the
    a2a summary (per-exchange bytes and GB/s against the per-direction link peak, the backend that
    ran, ranks seen) and a passing self-check (finite outputs, conserved tokens, gate gradient
    identical on every rank)."""
    import json
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), "--gpus", "8",
           "--steps", "3", "--warmup", "3", "--pipeline-n", "2", "--no-cpu-baseline", "--no-memory-sweep"]
    env = dict(os.environ, MPM_BENCH_BACKEND="gloo")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    line = [l_ for l_ in res.stdout.splitlines() if l_.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 8 and d["config"]["experts_per_gpu"] == 8
    assert d["self_check"]["ranks_seen"] == 8 and d["self_check"]["gate_grad_identical_across_ranks"]
    assert d["self_check"]["finite"] and d["self_check"]["tokens_conserved"]
    a2a = d["a2a"]
    assert a2a["backend"] == "p2p" and a2a["exchanges"], a2a
    assert all(x["remote_bytes"] > 0 for x in a2a["exchanges"])


@pytest.mark.parametrize("world,n,strategy", [(2, 2, "none"), (4, 3, "s4"), (2, 2, "s2")])
def test_step_graph_expert_parallel(tmp_path, world, n, strategy):
    """The whole expert-parallel step (flag waits, peer copy kernels, flag resets, the gate-gradient
    push + fixed-order sum) captured as one CUDA graph per rank and replayed three times: every
    replay is bit-identical to the eager step on the same inputs (stale or unreset flags would let a
    replay read rows before they land)."""
    d = _run(tmp_path, world, n, strategy, steps=1, graph=1)
    for r in range(world):
        assert int(d[f"r{r}_graph_replays_equal"]) == 3, r
    _check(d, world, n, steps=1)


def test_watchdog_aborts_on_stalled_peer(tmp_path):
    """Failure detection: rank 1 stalls after its forward, so rank 0's backward exchanges wait on flags
    that are never raised.  The exchange watchdog (csrc/watchdog.cu) must abort rank 0 with its
    diagnostic within the configured timeout instead of hanging the job."""
    import time
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "p2p_worker.py"),
           "--out", str(tmp_path / "x.npz"), "--chunks", "2", "--strategy", "none", "--stall-rank", "1"]
    env = dict(os.environ, MPM_WATCHDOG_TIMEOUT_S="5")
    t0 = time.monotonic()
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert res.returncode != 0
    assert "[mpm watchdog]" in res.stdout + res.stderr, (res.stdout + res.stderr)[-3000:]
    assert time.monotonic() - t0 < 200
