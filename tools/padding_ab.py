"""A/B of the capacity-padding skip (layer._skip_padding: valid_rows / valid_k at N = 1), interleaved
on the same layer and inputs: BASELINE configs[1] (cf 1.0) and configs[4]'s layer (128 experts top-1,
cf 1.25, 8K tokens), plus a skewed-gate variant of each.  Prints one JSON line per case.

  python tools/padding_ab.py [--reps 20] [--rounds 3]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200.layer import MoELayer  # noqa: E402

CASES = [("cfg2", 1024, 4096, 64, 2, 1.0, 16384), ("cfg5_layer", 1024, 4096, 128, 1, 1.25, 8192)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    for name, M, H, E, k, cf, T in CASES:
        for skew in (False, True):
            layer = MoELayer(M, H, E, top_k=k, capacity_factor=cf, pipeline=1, dtype=torch.bfloat16, device=dev)
            if skew:
                with torch.no_grad():
                    layer.gate_weight[: E // 4] *= 3.0
            g = torch.Generator(device=dev).manual_seed(0)
            x = torch.randn(T, M, device=dev, generator=g).bfloat16().requires_grad_(True)
            dy = torch.randn(T, M, device=dev, generator=g).bfloat16()

            def step():
                layer(x).backward(dy)
                x.grad = None
                for p in layer.parameters():
                    p.grad = None

            res = {True: [], False: []}
            for _ in range(args.rounds):
                for on in (True, False):
                    layer._skip_padding = on
                    layer.release_arenas()
                    for _ in range(3):
                        step()
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(args.reps):
                        step()
                    b.record()
                    torch.cuda.synchronize()
                    res[on].append(a.elapsed_time(b) / args.reps)
            kept = layer.last_arena.kept
            C = layer.last_arena.g.C
            fill = float(kept.sum()) / (E * C)
            on_ms, off_ms = statistics.median(res[True]), statistics.median(res[False])
            print(json.dumps({"case": name, "skewed_gate": skew, "capacity": C, "routed_fill": round(fill, 4),
                              "skip_ms": round(on_ms, 4), "noskip_ms": round(off_ms, 4),
                              "speedup": round(off_ms / on_ms, 4)}), flush=True)
            del layer


if __name__ == "__main__":
    main()
