"""Builds libmpm.so (the C-ABI of include/mpm.h) in-tree for sm_100a.

Plain nvcc, no torch headers: the library exposes only extern "C" entry
points over raw device pointers, so it loads with ctypes and links against
nothing but the CUDA runtime and the pip NCCL that torch already loads.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libmpm.so"
SOURCES = ["capi.cu", "routing.cu", "gate.cu", "gemm_simt.cu", "gemm_sm100.cu", "comm.cu", "p2p.cu", "clocks.cu", "watchdog.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[Path, Path]:
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    for root in roots:
        inc = Path(root) / "nccl" / "include"
        lib = Path(root) / "nccl" / "lib"
        if (inc / "nccl.h").exists() and (lib / "libnccl.so.2").exists():
            return inc, lib
    raise RuntimeError("pip NCCL (nvidia/nccl) not found; it ships with torch")


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _newer(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return False
    t = target.stat().st_mtime
    return all(d.stat().st_mtime <= t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    inc, lib = nccl_dirs()
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "mpm.h"]
    nvcc = _nvcc()
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{inc}",
                     "-Xptxas", "-v" if verbose else "-O3"]
    common += os.environ.get("MPM_NVCC_FLAGS", "").split()  # A/B builds (e.g. -DMPM_...=1)
    objs = []

    def compile_one(src: str) -> Path:
        s = CSRC / src
        o = BUILD / (s.stem + ".o")
        if not force and _newer(o, [s] + headers):
            return o
        cmd = [nvcc, *common, "-c", str(s), "-o", str(o)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        if verbose and res.stderr:
            sys.stderr.write(res.stderr)
        return o

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or not _newer(LIB, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), f"-L{lib}", "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={lib}"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
