"""A/B of the side-stream overlap in the backward (N = 1, BASELINE configs[1] shape): the gather
beside the deferred weight gradients on the gate stream, against running it after them on the
compute stream.  (An earlier variant also put the gate backward beside the expert backward: no
gain, since its tcgen05 GEMMs cannot share SMs with the persistent expert GEMMs; it now runs
serially ahead of them.)  Interleaved rounds
on one layer; per mode the median step time (no instrumentation) and the per-op device times of an
instrumented pass.  Prints one JSON line per mode.

  python tools/overlap_ab.py [--reps 20] [--rounds 3] [--experts 64] [--n 1]
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2506_22175_b200.layer import MoELayer  # noqa: E402

MODES = {"gather_side": True, "gather_serial": False}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--experts", type=int, default=64)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("--cool", type=float, default=2.0, help="idle seconds before each timed window")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    M, H, E, k, T = 1024, 4096, args.experts, 2, args.tokens
    layer = MoELayer(M, H, E, top_k=k, capacity_factor=1.0, pipeline=args.n, dtype=torch.bfloat16, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(T, M, device=dev, generator=g).bfloat16().requires_grad_(True)
    dy = torch.randn(T, M, device=dev, generator=g).bfloat16()

    def step():
        layer(x).backward(dy)
        x.grad = None
        for p in layer.parameters():
            p.grad = None

    res = {m: [] for m in MODES}
    clk = {m: [] for m in MODES}
    ops = {}
    for _ in range(args.rounds):
        for mode, gather in MODES.items():
            layer._gather_side = gather
            layer.record_times = False
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            time.sleep(args.cool)  # the step is power-capped under sustained load: time short windows
            sampler = ClockSampler(dev.index)
            sampler.start()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.monotonic()
            a.record()
            for _ in range(args.reps):
                step()
            b.record()
            torch.cuda.synchronize()
            w1 = time.monotonic()
            res[mode].append(a.elapsed_time(b) / args.reps)
            c = sampler.stop((w0, w1))
            clk[mode].append((c.get("sm_mhz"), c.get("reasons")))
            layer.record_times = True
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            ar = layer.last_arena
            fw, bw = ar.traces()
            ops[mode] = {"ops_ms": {e.op_id: round(e.duration * 1e3, 4) for tr in (fw, bw) for e in tr.events
                                    if e.duration > 0},
                         "wgrad_ms": round(ar.wgrad_seconds() * 1e3, 4), "phases_ms": ar.phase_ms()}
    for mode in MODES:
        print(json.dumps({"mode": mode, "experts": E, "tokens": T, "n": args.n,
                          "step_ms": round(statistics.median(res[mode]), 4),
                          "step_ms_all": [round(v, 4) for v in res[mode]], "clocks": clk[mode], **ops[mode]}), flush=True)


if __name__ == "__main__":
    main()
