"""BASELINE.json configs[4]: 12-layer Switch/BERT-MoE stack fwd+bwd step time.

N=1: `python tools/bench_stack.py`; N>1: `torchrun --nproc-per-node N tools/bench_stack.py`
(experts sharded E/N per GPU over the peer-memory exchanges; attention / LayerNorm /
gate parameters data parallel: their gradients are all-reduced inside the step, one
flattened NCCL all-reduce).

12 x (pre-LN attention + MoELayer: d_model 1024, d_ffn 4096, 128 experts
top-1, capacity 1.25), sequence 1024, batch `--batch` sequences per GPU
(default 8 -> 8K tokens/GPU).  A step = forward + backward
of the whole stack (synthetic bf16 input, random-init weights; the loss is
sum(y * dy) for a fixed random dy).  Prints one JSON line: step time,
tokens/s, the MoE layers' share of device time (per-layer CUDA events),
and peak memory.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2506_22175_b200.stack import MoEEncoder  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--pipeline-n", "--n", dest="n", default="1")  # under torchrun use --pipeline-n
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import os

    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("MPM_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
    pipeline = "adaptive" if args.n == "adaptive" else int(args.n)
    model = MoEEncoder(layers=args.layers, device=dev, pipeline=pipeline)
    D = 1024
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(args.batch, args.seq, D, device=dev, generator=g, dtype=torch.bfloat16)
    dy = torch.randn(args.batch, args.seq, D, device=dev, generator=g, dtype=torch.bfloat16)

    dense = [p for n_, p in model.named_parameters() if not (n_.endswith("moe.w1") or n_.endswith("moe.w2"))
             and not n_.endswith("moe.gate_weight")]

    def step():
        y = model(x)
        y.backward(dy)
        if world > 1:  # data-parallel dense parameters (the MoE layers reduce their own gate gradient)
            flat = torch.cat([p.grad.reshape(-1).float() for p in dense])
            dist.all_reduce(flat)
        for p in model.parameters():
            p.grad = None

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    # MoE share: one extra step with per-layer phase events
    for m in model.moe_layers():
        m.record_times = True
    step()  # builds timing arenas
    step()
    torch.cuda.synchronize()
    moe_ms = 0.0
    for m in model.moe_layers():
        ph = m.last_arena.phase_ms()
        moe_ms += ph["fwd_total"] + ph["bwd_total"]
    T = args.batch * args.seq
    if world > 1:
        t = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank != 0:
        if world > 1:
            dist.barrier()
        return
    print(json.dumps({"workload": f"{args.layers}-layer Switch/BERT-MoE encoder, d_model 1024, d_ffn 4096, "
                                  f"128 experts top-1 cf 1.25, seq {args.seq}, {T} tokens/GPU, bf16, N={world}",
                      "n_gpus": world, "tokens_per_s_all_gpus": world * T / (ms * 1e-3),
                      "ms_per_step": ms, "tokens_per_s": T / (ms * 1e-3),
                      "moe_layers_ms_per_step": moe_ms, "moe_share": moe_ms / ms,
                      "pipeline_n": args.n, "peak_memory_bytes": torch.cuda.max_memory_allocated(dev)}))
    if world > 1:
        dist.barrier()


if __name__ == "__main__":
    main()
