"""Worker for tests/test_gpu_p2p.py: one expert-parallel rank of MoELayer with
the peer-memory communicator (comm.PeerComm), launched by torchrun.

All ranks may share one GPU (CUDA IPC works across processes on the same
device), so the real multi-process path — IPC windows, copy-engine chunk
exchanges, stream-memory-op flag waits, the gate-gradient all-reduce — runs
on a single-GPU box.  torch.distributed uses gloo for the plumbing (handle
exchange, barriers); no byte of the layer moves through it.  Rank 0 gathers
every rank's inputs, weights, routing and results into an .npz for the test
to compare against the N-rank oracle.
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--chunks", default="2", help="pipeline n, or 'adaptive' (Algorithm 1, GPU-timed)")
    ap.add_argument("--strategy", default="none")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--T", type=int, default=512)
    ap.add_argument("--M", type=int, default=256)
    ap.add_argument("--H", type=int, default=512)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--cf", type=float, default=1.25)
    ap.add_argument("--graph", type=int, default=0, help="also capture a StepGraph and compare 3 replays")
    ap.add_argument("--skew", type=float, default=0.0,
                    help="gate bias toward experts 0 and 1 (skewed routing: drops there, empty experts elsewhere)")
    ap.add_argument("--stall-rank", type=int, default=-1,
                    help="this rank stops after its first forward (a stalled peer: the watchdog test)")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2506_22175_b200.layer import MoELayer

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ngpu)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    pipeline = "adaptive" if args.chunks == "adaptive" else int(args.chunks)
    layer = MoELayer(args.M, args.H, args.E, top_k=args.k, capacity_factor=args.cf, pipeline=pipeline,
                     memory_reuse=args.strategy, dtype=dtype, device=dev, candidates=(1, 2, 4))
    assert layer.comm.kind == "p2p", layer.comm
    if args.skew:  # the gate is replicated: every rank adds the same bias direction to the same rows
        with torch.no_grad():
            gen = torch.Generator().manual_seed(99)
            d_ = torch.randn(args.M, generator=gen)
            layer.gate_weight[:2] += (args.skew * d_ / d_.norm()).to(dev)
    g = torch.Generator().manual_seed(1000 + rank)
    results = []
    for step in range(args.steps):  # later steps reuse the arena: flags must have been reset
        x = torch.randn(args.T, args.M, generator=g).to(dtype).to(dev).requires_grad_(True)
        dy = torch.randn(args.T, args.M, generator=g).to(dtype).to(dev)
        mask = None
        if dtype == torch.bfloat16:  # this rank's ReLU mask (no-grad n=1 forward; pins the oracle's kink)
            with torch.no_grad():
                layer(x.detach(), n=1)
            a = layer.last_arena
            words = a.mask_full.view(a.g.e_loc, a.g.N * a.g.C, a.mask_w)[:, :, : a.g.H // 32].cpu().numpy()
            if a.compact:  # compacted expert side: source s's rows of expert e follow the lower sources'
                kept = a.win.tensor(a.wl.off["kept"], (a.g.N, a.g.E), torch.int32).cpu().numpy()
                cap = np.zeros_like(words)
                for el in range(a.g.e_loc):
                    e = rank * a.g.e_loc + el
                    o = 0
                    for s_ in range(a.g.N):
                        v = int(kept[s_, e])
                        cap[el, s_ * a.g.C: s_ * a.g.C + v] = words[el, o:o + v]
                        o += v
                words = cap
            mask = np.unpackbits(words.view(np.uint8), axis=-1, bitorder="little").astype(bool)
        y = layer(x)
        if rank == args.stall_rank:
            import time
            torch.cuda.synchronize()
            time.sleep(600)  # never joins the backward exchanges
        y.backward(dy)
        torch.cuda.synchronize()
        a = layer.last_arena
        results.append({k_: v.detach().float().cpu().numpy() for k_, v in dict(
            x=x, dy=dy, y=y, dx=x.grad, dwg=layer.gate_weight.grad, dw1=layer.w1.grad, dw2=layer.w2.grad,
            logits=a.logits, slot=a.slot, idx=a.idx).items()})
        if mask is not None:
            results[-1]["mask"] = mask
        for p in layer.parameters():
            p.grad = None
    graph_equal = -1
    if args.graph:  # the first step's inputs through a captured graph, replayed three times
        from paper_2506_22175_b200.spec import NO_REUSE, ReuseStrategy
        strat = NO_REUSE if args.strategy == "none" else ReuseStrategy.by_name(args.strategy)
        sg = layer.step_graph(args.T, int(args.chunks), strat)
        ref = results[0]
        graph_equal = 0
        for _ in range(3):
            y, (dx, dwg, dw1, dw2) = sg.replay(torch.from_numpy(ref["x"]).to(dtype).to(dev),
                                             torch.from_numpy(ref["dy"]).to(dtype).to(dev))
            torch.cuda.synchronize()
            got = dict(y=y, dx=dx, dwg=dwg, dw1=dw1, dw2=dw2)
            graph_equal += all(np.array_equal(v.float().cpu().numpy(), ref[k_]) for k_, v in got.items())
        sg.close()
    a = layer.last_arena
    state = dict(graph_replays_equal=graph_equal, compact=bool(getattr(a, "compact", False)),w1=layer.w1.detach().float().cpu().numpy(), w2=layer.w2.detach().float().cpu().numpy(),
                 wg=layer.gate_weight.detach().cpu().numpy(), results=results,
                 n=int(a.g.n), strategy=a.strategy.name if a.reuse else "none")
    gathered = [None] * world
    dist.all_gather_object(gathered, state)
    layer.release_arenas()  # collective window teardown
    layer.comm.close()
    if rank == 0:
        flat = {}
        for r, st in enumerate(gathered):
            for key in ("w1", "w2", "wg", "n", "strategy", "graph_replays_equal", "compact"):
                flat[f"r{r}_{key}"] = np.asarray(st[key])
            for s_, res in enumerate(st["results"]):
                for key, v in res.items():
                    flat[f"r{r}_s{s_}_{key}"] = v
        np.savez(args.out, **flat)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
