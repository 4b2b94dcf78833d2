"""Per-GPU compute of BASELINE configs[1] at N=8, on one GPU: the layer with the
8 local experts an N=8 rank owns (E=8, each receiving 8 x 512 = 4096 rows at
T=16K, k=2, cf 1.0) — everything of the N=8 step except the NVLink exchange.
Times the fwd+bwd step (CUDA events, eager autograd path like bench.py) for
n in {1, 2, 4, 8} and reuse none / S4, so the chunking overhead the N=8
pipeline pays to hide its all-to-all is measured, not modelled."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402

dev = torch.device("cuda", 0)
T, M, H, E, k = 16384, 1024, 4096, 8, 2
layer = MoELayer(M, H, E, top_k=k, capacity_factor=1.0, pipeline=1, dtype=torch.bfloat16, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, M, device=dev, generator=g).bfloat16().requires_grad_(True)
dy = torch.randn(T, M, device=dev, generator=g).bfloat16()
flops = 12.0 * k * M * H * T  # expert FLOPs per step


def step(n, strat):
    y = layer(x, n=n, strategy=strat)
    y.backward(dy)
    x.grad = None
    for p in layer.parameters():
        p.grad = None


out = []
for strat in (None, "s4"):
    for n in (1, 2, 4, 8):
        for _ in range(4):
            step(n, strat)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        time.sleep(1.0)  # power-limited part: every configuration starts its window from idle
        a.record()
        for _ in range(reps):
            step(n, strat)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        rec = {"n": n, "strategy": strat or "none", "ms_per_step": round(ms, 4),
               "tokens_per_s": round(T / ms * 1e3), "expert_tflops": round(flops / ms / 1e9, 1)}
        if "--detail" in sys.argv:  # one instrumented step: per-op device time, phases
            layer.record_times = True
            step(n, strat)
            step(n, strat)
            torch.cuda.synchronize()
            ar = layer.last_arena
            fw, bw = ar.traces()
            ops_ms = {}
            for tr in (fw, bw):
                for e in tr.events:
                    key = e.op_id.split("_")[0] if "_" in e.op_id else e.op_id.rstrip("0123456789")
                    ops_ms[key] = round(ops_ms.get(key, 0.0) + e.duration * 1e3, 4)
            rec.update({"fwd_span_ms": round(fw.makespan * 1e3, 4), "bwd_span_ms": round(bw.makespan * 1e3, 4),
                        "op_sum_ms": ops_ms, "wgrad_ms": round(ar.wgrad_seconds() * 1e3, 4),
                        "phases_ms": ar.phase_ms()})
            layer.record_times = False
        out.append(rec)
        print(json.dumps(rec), flush=True)
        layer.release_arenas()
