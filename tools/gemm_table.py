"""Per-GEMM table: the six expert GEMMs of the layer at BASELINE configs[1] (N=1: 64 local experts x 512
capacity rows) and at the N=8 per-GPU shape (8 local experts x 4096 rows), in the layouts and epilogues
the layer issues them with (layer.py _calls), next to cuBLAS (torch.bmm on the same operands, plain
epilogue).  CUDA events, L2 flushed (a 512 MiB write) before every timed repetition.  Prints one JSON
line per shape; `--out` writes the list.

--sustained adds a steady-state measurement: each GEMM back to back for ~40 ms (the layer step's regime)
with the in-kernel SM clock trace (mpm_clock_trace), so each GEMM's time is reported with the SM clock
it ran at and as TFLOP/s normalised to the maximum clock (the B200 is power-limited under these
kernels: the clock drops well below its maximum within ~1 ms).

  python tools/gemm_table.py [--reps 20] [--sustained] [--out profiles/r2_gemm_vs_cublas.json]
"""
import ctypes
import time
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(0)
flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def bf(*s):
    return (torch.randn(*s, device=dev, generator=gen) * 0.1).bfloat16()


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush_buf.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps * 1e-3


_nvml = None


def _energy_mj():
    """Board energy counter (mJ) from NVML, or None."""
    global _nvml
    try:
        import pynvml
        if _nvml is None:
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(dev)
            _nvml = pynvml.nvmlDeviceGetHandleByPciBusId(
                f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        return float(pynvml.nvmlDeviceGetTotalEnergyConsumption(_nvml))
    except Exception:
        return None


def sustained(fn, ms_target=40.0, interval_us=5.0, energy=False):
    """Steady state of `fn` run back to back: (seconds per launch, effective SM MHz[, joules per
    launch]).  The time (and NVML board energy, over ~10x ms_target so the counter's few-ms update
    granularity does not matter) come from an untraced run; the SM clock from a second run with the
    in-kernel clock tracer, whose own time is returned in `traced_s` so a disturbed trace shows."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    reps = max(5, int(ms_target / max(a.elapsed_time(b), 1e-3)))
    # untraced: time and energy
    reps_e = reps * (10 if energy else 1)
    time.sleep(0.5)
    e0 = _energy_mj() if energy else None
    a.record()
    for _ in range(reps_e):
        fn()
    b.record()
    torch.cuda.synchronize()
    e1 = _energy_mj() if energy else None
    per = a.elapsed_time(b) * 1e-3 / reps_e
    joules = (e1 - e0) * 1e-3 / reps_e if e0 is not None and e1 is not None else None
    # traced: the SM clock
    n = int(ms_target * 1.5e3 / interval_us) + 1000
    buf = torch.zeros(2 * n, dtype=torch.int64, device=dev)
    side = torch.cuda.Stream(device=dev)
    time.sleep(0.5)
    _lib.call("mpm_clock_trace", ctypes.c_void_p(buf.data_ptr()), n, int(interval_us * 1000),
              ctypes.c_void_p(side.cuda_stream))
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    tr = buf.view(n, 2).cpu().tolist()
    win = [r for r in tr if 0 < r[0] and r[0] - tr[0][0] <= ms * 1e6]
    mhz = (win[-1][1] - win[0][1]) / (win[-1][0] - win[0][0]) * 1e3
    return per, mhz, joules, ms * 1e-3 / reps


def shapes(E, R, M, H):
    """(name, batches, rows, N, K, a_mn, b_mn, epilogue) of the six expert GEMMs (layer.py _calls)."""
    return [
        ("fc1_fwd", E, R, H, M, False, False, "relu_mask"),
        ("fc2_fwd", E, R, M, H, False, False, "none"),
        ("fc2_dgrad", E, R, H, M, False, True, "dmask"),
        ("fc1_dgrad", E, R, M, H, False, True, "none"),
        ("fc2_wgrad", E, M, H, R, True, True, "none"),
        ("fc1_wgrad", E, H, M, R, True, True, "none"),
    ]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--sustained", action="store_true")
    ap.add_argument("--only", default=None, help="cfg2_N1 or cfg2_N8_per_gpu")
    ap.add_argument("--gemm", default=None, help="comma list of GEMM names")
    args = ap.parse_args()
    M, H = 1024, 4096
    rows = []
    for label, E, R in (("cfg2_N1", 64, 512), ("cfg2_N8_per_gpu", 8, 4096)):
        if args.only and args.only != label:
            continue
        for name, B, Rw, N, K, amn, bmn, epi in shapes(E, R, M, H):
            if args.gemm and name not in args.gemm.split(","):
                continue
            a = bf(B, K, Rw) if amn else bf(B, Rw, K)
            b = bf(B, K, N) if bmn else bf(B, N, K)
            c = torch.empty(B, Rw, N, device=dev, dtype=torch.bfloat16)
            mask = torch.zeros(B, Rw, N // 32, device=dev, dtype=torch.int32)
            code = {"relu_mask": _lib.EPI_RELU_MASK, "dmask": _lib.EPI_DMASK, "none": _lib.EPI_NONE}[epi]
            aux = mask if epi != "none" else None
            t = timeit(lambda: ops.gemm(a, b, c, a_mn_major=amn, b_mn_major=bmn, epilogue=code, aux=aux), args.reps)
            A = a.transpose(1, 2) if amn else a
            Bt = b if bmn else b.transpose(1, 2)
            tc = timeit(lambda: torch.bmm(A, Bt, out=c), args.reps)
            f = 2.0 * B * Rw * N * K
            row = {"shape": label, "gemm": name, "batches": B, "rows": Rw, "n": N, "k": K, "a_mn": amn, "b_mn": bmn,
                   "epilogue": epi, "ours_us": t * 1e6, "ours_tflops": f / t / 1e12,
                   "cublas_us": tc * 1e6, "cublas_tflops": f / tc / 1e12, "ours_over_cublas": tc / t}
            if args.sustained:
                fmax = 1965.0
                for tag, fn_ in (("ours", lambda: ops.gemm(a, b, c, a_mn_major=amn, b_mn_major=bmn, epilogue=code,
                                                           aux=aux)),
                                 ("cublas", lambda: torch.bmm(A, Bt, out=c))):
                    ts, mhz, jl, traced = sustained(fn_, energy=True)
                    row[f"{tag}_traced_us"] = traced * 1e6
                    row[f"{tag}_sustained_mj_per_launch"] = jl * 1e3 if jl is not None else None
                    row[f"{tag}_sustained_pj_per_flop"] = jl / f * 1e12 if jl is not None else None
                    row[f"{tag}_sustained_us"] = ts * 1e6
                    row[f"{tag}_sustained_mhz"] = round(mhz, 1)
                    row[f"{tag}_sustained_tflops"] = f / ts / 1e12
                    row[f"{tag}_sustained_tflops_at_max_clock"] = f / ts / 1e12 * fmax / mhz
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1) + "\n")


if __name__ == "__main__":
    main()
