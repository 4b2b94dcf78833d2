"""ctypes binding of libmpm.so (the C-ABI declared in include/mpm.h).

The product path has no fallback: if the library is missing or fails to
load, every op raises MpmLibraryError.  Tests that only need the exported
symbol table (no GPU) call `load()` directly.
"""

from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libmpm.so"
HEADER = PKG.parent / "include" / "mpm.h"

MPM_F32 = 0
MPM_BF16 = 1

EPI_NONE, EPI_RELU, EPI_DRELU, EPI_STORE_F32, EPI_ACCUM_F32, EPI_ADD_AUX_F32, EPI_RELU_MASK, EPI_DMASK, EPI_ACCUM = range(9)
A2A_DISPATCH, A2A_COMBINE = 0, 1
COPY_D2H, COPY_H2D, COPY_D2D = 0, 1, 2


class MpmLibraryError(RuntimeError):
    """libmpm.so is missing / unloadable — there is no CPU fallback."""


class MpmError(RuntimeError):
    """A C-ABI call returned a nonzero status."""

    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed with status {status}: {msg}")
        self.status = status


class GemmArgs(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int),
        ("epilogue", ctypes.c_int),
        ("batches", ctypes.c_int64),
        ("rows", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("k", ctypes.c_int64),
        ("a", ctypes.c_void_p), ("a_ld", ctypes.c_int64), ("a_batch_stride", ctypes.c_int64),
        ("a_mn_major", ctypes.c_int),
        ("b", ctypes.c_void_p), ("b_ld", ctypes.c_int64), ("b_batch_stride", ctypes.c_int64),
        ("b_mn_major", ctypes.c_int),
        ("c", ctypes.c_void_p), ("c_ld", ctypes.c_int64), ("c_batch_stride", ctypes.c_int64),
        ("c_dtype", ctypes.c_int),
        ("aux", ctypes.c_void_p), ("aux_ld", ctypes.c_int64), ("aux_batch_stride", ctypes.c_int64),
        ("valid_rows", ctypes.c_void_p),
        ("a_k_period", ctypes.c_int64), ("b_k_period", ctypes.c_int64),
        ("k_splits", ctypes.c_int64), ("split_stride", ctypes.c_int64),
        ("valid_k", ctypes.c_void_p),
    ]


MAX_PEERS = 64
IPC_HANDLE_BYTES = 64


class P2PCopy(ctypes.Structure):
    _fields_ = [("dst", ctypes.c_void_p), ("src", ctypes.c_void_p), ("dpitch", ctypes.c_int64),
                ("spitch", ctypes.c_int64), ("width", ctypes.c_int64), ("height", ctypes.c_int64)]


class PushPlan(ctypes.Structure):
    """mpm_push_plan: the fused dispatch of one chunk from this rank to every destination."""
    _fields_ = [("nranks", ctypes.c_int), ("rank", ctypes.c_int),
                ("dst", ctypes.c_void_p * MAX_PEERS), ("flag", ctypes.c_void_p * MAX_PEERS),
                ("e_loc", ctypes.c_int64), ("capacity", ctypes.c_int64), ("e0", ctypes.c_int64),
                ("ne", ctypes.c_int64), ("s0", ctypes.c_int64), ("cs", ctypes.c_int64),
                ("x_stride", ctypes.c_int64), ("x_row0", ctypes.c_int64), ("counter", ctypes.c_void_p),
                ("kept_all", ctypes.c_void_p)]


class P2PPlan(ctypes.Structure):
    """mpm_p2p_plan: waits -> one SM copy kernel (raises the peer flags) -> arrival waits -> resets."""
    _fields_ = [("n_wait", ctypes.c_int), ("wait", ctypes.c_void_p * MAX_PEERS),
                ("n_copy", ctypes.c_int), ("copy", P2PCopy * MAX_PEERS),
                ("n_signal", ctypes.c_int), ("signal", ctypes.c_void_p * MAX_PEERS),
                ("n_arrive", ctypes.c_int), ("arrive", ctypes.c_void_p * MAX_PEERS),
                ("n_reset", ctypes.c_int), ("reset", ctypes.c_void_p * MAX_PEERS),
                ("counter", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_S = ctypes.c_size_t

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "mpm_abi_version": [],
    "mpm_last_error": [],
    "mpm_sm_count": [],
    "mpm_launch_count": [],
    "mpm_gate_fwd": [_P, _I, _P, _P, _L, _L, _L, _P, _P],
    "mpm_gate_workspace_bytes": [_L, _L, _L],
    "mpm_route_workspace_bytes": [_L, _L, _I],
    "mpm_route": [_P, _L, _L, _I, _I, _P, _P, _P, _P],
    "mpm_gate_route": [_P, _I, _P, _L, _L, _L, _I, _I, _P, _P, _P, _P, _P, _P],
    "mpm_assign_slots": [_P, _L, _L, _I, _L, _P, _P, _P, _P],
    "mpm_chunk_rows": [_P, _L, _L, _I, _P, _P],
    "mpm_permute": [_P, _I, _P, _P, _P, _L, _L, _L, _I, _L, _I, _P, _P],
    "mpm_combine": [_P, _I, _P, _P, _P, _L, _L, _L, _I, _L, _I, _P, _P],
    "mpm_combine_bwd": [_P, _P, _I, _P, _P, _P, _P, _L, _L, _L, _I, _L, _I, _P, _P, _P],
    "mpm_gate_bwd_logits": [_P, _P, _P, _P, _L, _L, _I, _I, _P, _P],
    "mpm_gather_bwd": [_P, _I, _P, _P, _P, _P, _L, _L, _L, _I, _L, _I, _P, _P, _P],
    "mpm_gate_wgrad": [_P, _P, _I, _L, _L, _L, _P, _P, _P],
    "mpm_gate_backward": [_P, _P, _P, _P, _P, _P, _P, _I, _P, _L, _L, _L, _I, _I, _L, _I, _P, _P, _P, _P, _P],
    "mpm_gate_backward_gate": [_P, _P, _P, _P, _P, _I, _P, _L, _L, _L, _I, _I, _P, _P, _P, _P, _P],
    "mpm_gate_backward_gather": [_P, _I, _P, _P, _P, _P, _L, _L, _L, _I, _L, _I, _P, _P, _P],
    "mpm_combine_bwd_gate": [_P, _P, _I, _P, _P, _P, _P, _P, _L, _L, _L, _I, _I, _L, _I, _P, _P, _P, _P, _P],
    "mpm_gate_backward_gemms": [_P, _I, _P, _P, _L, _L, _L, _I, _I, _P, _P, _P, _P],
    "mpm_gate_gather": [_P, _I, _P, _P, _P, _P, _L, _L, _L, _I, _I, _L, _I, _P, _P, _P],
    "mpm_clock_trace": [_P, _I, _L, _P],
    "mpm_grouped_gemm": [ctypes.POINTER(GemmArgs), _P],
    "mpm_grouped_gemm_simt": [ctypes.POINTER(GemmArgs), _P],
    "mpm_splitk_reduce": [_P, _L, _L, _L, _P, _I, _I, _P],
    "mpm_comm_unique_id": [_P],
    "mpm_comm_init": [_P, _I, _I, _I, ctypes.POINTER(ctypes.c_void_p)],
    "mpm_comm_destroy": [_P],
    "mpm_a2a_chunk": [_P, _I, _I, _P, _P, _P, _L, _I, _P, _P, _P],
    "mpm_copy_async": [_P, _P, _S, _I, _P],
    "mpm_ipc_alloc": [_S, ctypes.POINTER(ctypes.c_void_p), _P],
    "mpm_ipc_open": [_P, ctypes.POINTER(ctypes.c_void_p)],
    "mpm_ipc_close": [_P],
    "mpm_ipc_free": [_P],
    "mpm_p2p_run": [ctypes.POINTER(P2PPlan), ctypes.c_uint32, _P],
    "mpm_sum_slices": [_P, _I, _L, _L, _P, _P],
    "mpm_watchdog_watch": [_P, ctypes.c_double, ctypes.c_char_p],
    "mpm_dispatch_push": [ctypes.POINTER(PushPlan), _P, _I, _L, _I, _P, _P, ctypes.c_uint32, _P],
    "mpm_slot_owners": [_P, _P, _P, _L, _L, _I, _L, _P, _P],
    "mpm_combine_push": [ctypes.POINTER(PushPlan), _P, _I, _L, ctypes.c_uint32, _P],
    "mpm_compact_rows": [_P, _I, _L, _L, _I, _L, _L, _P, _P],
    "mpm_compact_pull": [ctypes.POINTER(PushPlan), _P, _I, _L, _P],
    "mpm_watchdog_pending": [],
    "mpm_watchdog_fired": [],
    "mpm_event_create": [_I, ctypes.POINTER(ctypes.c_void_p)],
    "mpm_event_destroy": [_P],
    "mpm_event_record": [_P, _P],
    "mpm_stream_wait": [_P, _P],
    "mpm_event_elapsed_ms": [_P, _P, ctypes.POINTER(ctypes.c_float)],
    "mpm_clock_sampler_start": [ctypes.c_char_p, _I],
    "mpm_clock_sampler_stop": [ctypes.POINTER(ctypes.c_double), _I, ctypes.POINTER(ctypes.c_int)],
    "mpm_monotonic": [],
}
_RESTYPES = {"mpm_last_error": ctypes.c_char_p, "mpm_route_workspace_bytes": ctypes.c_size_t,
             "mpm_gate_workspace_bytes": ctypes.c_size_t, "mpm_launch_count": ctypes.c_ulonglong,
             "mpm_watchdog_fired": ctypes.c_ulonglong,
             "mpm_monotonic": ctypes.c_double}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares (the export contract)."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|size_t|const char\*|unsigned long long)\s+(mpm_\w+)\s*\(", text, re.M)))


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("MPM_LIB", LIB_PATH))
    if not path.exists():
        raise MpmLibraryError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA extension is required; there is no CPU fallback)")
    try:
        lib = ctypes.CDLL(str(path))
    except OSError as exc:  # pragma: no cover - environment specific
        raise MpmLibraryError(f"cannot load {path}: {exc}") from exc
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = lib
    return lib


def launch_count() -> int:
    """Kernels libmpm launched so far in this process (counted in C at every launch site)."""
    return int(load().mpm_launch_count())


def call(name: str, *args) -> int:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.mpm_last_error().decode(errors="replace")
        raise MpmError(name, rc, msg)
    return rc


class Call:
    """One prebuilt C-ABI call: fn(*args), raising MpmError on a nonzero status.

    Arguments are converted once; mutable ctypes objects in `args` (stream
    handles, pointers) may be updated in place between issues.
    """

    __slots__ = ("name", "fn", "args")

    def __init__(self, name: str, *args) -> None:
        self.name = name
        self.fn = getattr(load(), name)
        self.args = args

    def __call__(self) -> None:
        rc = self.fn(*self.args)
        if rc != 0:
            raise MpmError(self.name, rc, load().mpm_last_error().decode(errors="replace"))


class Event:
    """A raw CUDA event owned through the C-ABI."""

    __slots__ = ("handle", "timing")

    def __init__(self, timing: bool = False) -> None:
        self.handle = ctypes.c_void_p()
        self.timing = timing
        call("mpm_event_create", int(timing), ctypes.byref(self.handle))

    def record(self, stream) -> None:
        call("mpm_event_record", self.handle, stream)

    def elapsed_ms(self, end: "Event") -> float:
        out = ctypes.c_float()
        call("mpm_event_elapsed_ms", self.handle, end.handle, ctypes.byref(out))
        return float(out.value)

    def __del__(self):  # pragma: no cover - teardown order varies
        try:
            if self.handle:
                load().mpm_event_destroy(self.handle)
        except Exception:
            pass


def stream_wait(stream, event: Event) -> None:
    call("mpm_stream_wait", stream, event.handle)
