"""Compacted vs capacity expert side at N > 1 (run under torchrun; ranks may share one GPU for a
functional/relative measurement): fwd+bwd step time (max over ranks, median of interleaved rounds)
of one layer with MPM_COMPACT on and off in the same processes.

  torchrun --nproc-per-node 2 tools/compact_probe.py [--E 128 --k 1 --cf 1.25 --T 8192 --n 1]
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402
from paper_2506_22175_b200.spec import NO_REUSE  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=1024)
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--E", type=int, default=128)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--cf", type=float, default=1.25)
    ap.add_argument("--T", type=int, default=8192)
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("--rounds", type=int, default=5)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    layers = {}
    for mode in ("1", "0"):
        lay = MoELayer(args.M, args.H, args.E, top_k=args.k, capacity_factor=args.cf, pipeline=args.n,
                       dtype=torch.bfloat16, device=dev)
        lay._compact = mode == "1"
        layers[mode] = lay
    g = torch.Generator().manual_seed(rank)
    x = torch.randn(args.T, args.M, generator=g).bfloat16().to(dev)
    dy = torch.randn(args.T, args.M, generator=g).bfloat16().to(dev)

    def step_ms(lay, reps=5):
        lay.run_step(x, dy, args.n, NO_REUSE)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            lay.run_step(x, dy, args.n, NO_REUSE)
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    res = {"1": [], "0": []}
    for _ in range(args.rounds):
        for mode in ("1", "0"):
            res[mode].append(step_ms(layers[mode]))
    a = layers["1"].last_arena
    kept = a.kept.float()
    pad = 1.0 - float(kept.sum()) / (a.g.E * a.g.C)
    if rank == 0:
        print(json.dumps({"config": vars(args), "world": world, "compact_active": bool(a.compact),
                          "padding_fraction_rank0": round(pad, 4),
                          "ms_compact": statistics.median(res["1"]), "ms_capacity": statistics.median(res["0"]),
                          "rounds": res}), flush=True)
    for lay in layers.values():
        lay.release_arenas()
        lay.comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
