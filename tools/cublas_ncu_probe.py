"""Run the six expert GEMMs of BASELINE configs[1] (N=1 and N=8 per-GPU shapes) once each through
cuBLAS (torch.bmm) and once through libmpm, for an ncu capture that compares the two on the same
counters: kernel name (cuBLAS encodes its tile / cluster shape there), tensor-pipe active %, L2->SM
sectors, DRAM bytes, SM clock.

  ncu --set full --clock-control none -k regex:"nvjet|gemm|umma" -o gpurun_out/cublas_vs_ours \
      python tools/cublas_ncu_probe.py [--only cfg2_N1]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_22175_b200 import _lib, ops  # noqa: E402
from tools.gemm_table import shapes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--impl", default="both", choices=["both", "ours", "cublas"])
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(0)
    M, H = 1024, 4096
    for label, E, R in (("cfg2_N1", 64, 512), ("cfg2_N8_per_gpu", 8, 4096)):
        if args.only and args.only != label:
            continue
        for name, B, Rw, N, K, amn, bmn, epi in shapes(E, R, M, H):
            a = ((torch.randn(B, K, Rw, device=dev, generator=gen) if amn
                  else torch.randn(B, Rw, K, device=dev, generator=gen)) * 0.1).bfloat16()
            b = ((torch.randn(B, K, N, device=dev, generator=gen) if bmn
                  else torch.randn(B, N, K, device=dev, generator=gen)) * 0.1).bfloat16()
            c = torch.empty(B, Rw, N, device=dev, dtype=torch.bfloat16)
            mask = torch.zeros(B, Rw, N // 32, device=dev, dtype=torch.int32)
            code = {"relu_mask": _lib.EPI_RELU_MASK, "dmask": _lib.EPI_DMASK, "none": _lib.EPI_NONE}[epi]
            A = a.transpose(1, 2) if amn else a
            Bt = b if bmn else b.transpose(1, 2)
            if args.impl in ("both", "ours"):
                ops.gemm(a, b, c, a_mn_major=amn, b_mn_major=bmn, epilogue=code, aux=mask if epi != "none" else None)
            if args.impl in ("both", "cublas"):
                torch.bmm(A, Bt, out=c)
            torch.cuda.synchronize()
            print(label, name, flush=True)


if __name__ == "__main__":
    main()
