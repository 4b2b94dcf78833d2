"""Expert-parallel communicators for the chunk all-to-alls.

PeerComm (the default for N > 1): exchanges over NVLink peer memory.  Each
step arena exports one device window through CUDA IPC (handles exchanged
with torch.distributed, any backend); chunk exchanges are prebuilt
mpm_p2p_run plans (csrc/p2p.cu): pulls for dispatch-type ops, pushes +
flags for combine-type ops, one light copy kernel each (it fits beside the
persistent GEMM CTAs) and no host synchronisation.

ExpertComm ("nccl"): the baseline — grouped ncclSend/ncclRecv through a
libmpm-owned NCCL communicator (unique id broadcast through
torch.distributed).

With one rank (or no process group) nothing is created: the chunk
all-to-alls degenerate to identities (PAPER.md:520 / SURVEY.md §8e).
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .ops import _p, _s, dtype_code


def block_plan(direction: int, nranks: int, e_loc: int, c_i: int, width: int, capacity: int, s_i: int,
               x_stride: int, x_row0: int, e0: int = 0, ne: int | None = None
               ) -> tuple[list[int], list[int], list[int]]:
    """(peer, send offset, recv offset) in elements per block of c_i*width elements, for the chunk of
    local experts [e0, e0+ne) (default: all) and capacity slots [s_i, s_i+c_i).

    Source side (dispatch): this rank's expert-major buffer [E][C][W]; the
    block for (peer d, local expert el) is rows [(d*E_loc+el)*C + s_i, +c_i).
    Expert side: expert el's rows start at (el-e0)*x_stride + x_row0,
    source-major (source s at + s*c_i); x_row0 is the row of (expert e0,
    source 0, slot s_i).  A full (all-chunk) buffer uses x_stride = N*C,
    x_row0 = e0*N*C + N*s_i; a per-chunk ring slot x_stride = N*c_i,
    x_row0 = 0.  Combine is the inverse.  Blocks are ordered (peer, el) on
    every rank, so the b-th send to a peer pairs with that peer's b-th
    receive from this rank.
    """
    ne = e_loc - e0 if ne is None else ne
    peers, send, recv = [], [], []
    for peer in range(nranks):
        for el in range(e0, e0 + ne):
            source = ((peer * e_loc + el) * capacity + s_i) * width
            expert = ((el - e0) * x_stride + x_row0 + peer * c_i) * width
            peers.append(peer)
            if direction == _lib.A2A_DISPATCH:
                send.append(source)
                recv.append(expert)
            else:
                send.append(expert)
                recv.append(source)
    return peers, send, recv


class ExpertComm:
    kind = "nccl"

    def __init__(self, group=None, device: torch.device | None = None) -> None:
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.nranks = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.nranks, self.rank = 1, 0
        self.handle = None
        self.device = device
        if self.nranks > 1:
            self._init_nccl()

    def _init_nccl(self) -> None:
        buf = (ctypes.c_char * 128)()
        if self.rank == 0:
            _lib.call("mpm_comm_unique_id", ctypes.cast(buf, ctypes.c_void_p))
        obj = [bytes(buf) if self.rank == 0 else None]
        src = dist.get_global_rank(self.group, 0) if self.group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=self.group)
        uid = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        dev = (self.device or torch.device("cuda", torch.cuda.current_device())).index or 0
        handle = ctypes.c_void_p()
        _lib.call("mpm_comm_init", ctypes.cast(uid, ctypes.c_void_p), self.nranks, self.rank, dev,
                  ctypes.byref(handle))
        self.handle = handle

    def a2a(self, direction: int, src: torch.Tensor, dst: torch.Tensor, plan, block: int, stream=None) -> None:
        """Run one chunk's block plan (see block_plan) between two base buffers."""
        peers, soff, roff = plan
        n = len(peers)
        _lib.call("mpm_a2a_chunk", self.handle, self.nranks, n, (ctypes.c_int32 * n)(*peers),
                  (ctypes.c_int64 * n)(*soff), (ctypes.c_int64 * n)(*roff), block,
                  dtype_code(src.dtype), _p(src), _p(dst), _s(stream))

    def all_reduce(self, t: torch.Tensor) -> None:
        dist.all_reduce(t, group=self.group)

    def close(self) -> None:
        if self.handle is not None:
            _lib.call("mpm_comm_destroy", self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order varies
        try:
            self.close()
        except Exception:
            pass


class LoopbackHub:
    """Shared state of LoopbackComm ranks living in one process (one GPU).

    Test infrastructure for the N > 1 data path on a single device: each
    rank's layer is driven by its own host thread and its own CUDA streams;
    an exchange publishes every rank's send buffer and stream event, then each
    rank pulls its blocks with device copies on its own stream, exactly as the
    block plan pairs them (b-th send to a peer <-> that peer's b-th receive).
    """

    def __init__(self, world: int) -> None:
        import threading

        self.world = world
        self.barrier = threading.Barrier(world, timeout=120)  # a stuck rank fails loudly, never hangs
        self.slots: dict = {}


class LoopbackComm:
    """ExpertComm stand-in for `world` ranks sharing one GPU (see LoopbackHub)."""

    loopback = True
    handle = None

    def __init__(self, hub: LoopbackHub, rank: int) -> None:
        self.hub, self.rank, self.nranks = hub, rank, hub.world

    def _publish(self, item) -> dict:
        self.hub.barrier.wait()          # previous exchange fully consumed
        self.hub.slots[self.rank] = item
        self.hub.barrier.wait()
        return dict(self.hub.slots)

    def a2a(self, direction: int, src: torch.Tensor, dst: torch.Tensor, plan, block: int, stream=None) -> None:
        stream = stream or torch.cuda.current_stream()
        ready = torch.cuda.Event()
        ready.record(stream)
        slots = self._publish((src, ready, plan))
        peers, _, roff = plan
        for p in range(self.nranks):
            psrc, pready, pplan = slots[p]
            stream.wait_event(pready)
            sends = [so for pp, so in zip(pplan[0], pplan[1]) if pp == self.rank]
            recvs = [ro for pp, ro in zip(peers, roff) if pp == p]
            with torch.cuda.stream(stream):
                for so, ro in zip(sends, recvs):
                    dst.view(-1)[ro:ro + block].copy_(psrc.view(-1)[so:so + block], non_blocking=True)
        done = torch.cuda.Event()
        done.record(stream)
        slots = self._publish(done)
        for p in range(self.nranks):  # senders may reuse their buffers only after every pull
            stream.wait_event(slots[p])

    def all_reduce(self, t: torch.Tensor) -> None:
        stream = torch.cuda.current_stream()
        ready = torch.cuda.Event()
        ready.record(stream)
        slots = self._publish((t.clone(), ready))
        for p in range(self.nranks):
            stream.wait_event(slots[p][1])
        total = slots[0][0].clone()
        for p in range(1, self.nranks):  # fixed rank order: identical sums on every rank
            total += slots[p][0]
        t.copy_(total)
        done = torch.cuda.Event()
        done.record(stream)
        for ev in self._publish(done).values():
            stream.wait_event(ev)

    def close(self) -> None:
        pass


# ------------------------------------------------------------------ p2p
class _CudaArray:
    """__cuda_array_interface__ over raw device bytes (torch.as_tensor adopts it without a copy)."""

    def __init__(self, ptr: int, nbytes: int) -> None:
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": (nbytes,), "typestr": "|u1",
                                         "version": 3, "strides": None}


class Window:
    """One rank's IPC-exported device window plus every peer's mapping of theirs.

    Collective: every rank of the group creates its windows in the same
    order with the same size (the arenas are rank-symmetric), so an object
    at byte offset `off` lives at `addr(r, off)` in rank r's window.
    """

    def __init__(self, comm: "PeerComm", nbytes: int) -> None:
        self.comm, self.nbytes = comm, int(nbytes)
        ptr = ctypes.c_void_p()
        handle = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
        _lib.call("mpm_ipc_alloc", self.nbytes, ctypes.byref(ptr), ctypes.cast(handle, ctypes.c_void_p))
        self.local = int(ptr.value)
        handles = [None] * comm.nranks
        dist.all_gather_object(handles, bytes(handle), group=comm.group)
        self.bases: list[int] = []
        for r, h in enumerate(handles):
            if r == comm.rank:
                self.bases.append(self.local)
                continue
            p = ctypes.c_void_p()
            hb = (ctypes.c_char * _lib.IPC_HANDLE_BYTES).from_buffer_copy(h)
            _lib.call("mpm_ipc_open", ctypes.cast(hb, ctypes.c_void_p), ctypes.byref(p))
            self.bases.append(int(p.value))
        dist.barrier(group=comm.group)  # every mapping exists before any peer touches it
        dev = comm.device or torch.device("cuda", torch.cuda.current_device())
        self._bytes = torch.as_tensor(_CudaArray(self.local, self.nbytes), device=dev)

    def addr(self, rank: int, offset: int) -> int:
        return self.bases[rank] + int(offset)

    def tensor(self, offset: int, shape, dtype: torch.dtype) -> torch.Tensor:
        """A view of this rank's window bytes [offset, offset + numel*size) as `dtype`."""
        numel = 1
        for d in shape:
            numel *= int(d)
        nbytes = numel * torch.empty((), dtype=dtype).element_size()
        return self._bytes[offset:offset + nbytes].view(dtype).view(*shape)

    def close(self) -> None:
        """Collective: unmap the peers' windows, then free this one."""
        if self.local is None:
            return
        torch.cuda.synchronize()
        dist.barrier(group=self.comm.group)  # nobody copies from / into a window any more
        for r, b in enumerate(self.bases):
            if r != self.comm.rank:
                _lib.call("mpm_ipc_close", ctypes.c_void_p(b))
        dist.barrier(group=self.comm.group)
        self._bytes = None
        _lib.call("mpm_ipc_free", ctypes.c_void_p(self.local))
        self.local = None


class PeerComm:
    """Chunk exchanges over peer memory (csrc/p2p.cu); see the module doc."""

    kind = "p2p"
    handle = None

    def __init__(self, group=None, device: torch.device | None = None) -> None:
        if not (dist.is_available() and dist.is_initialized()):
            raise RuntimeError("PeerComm needs an initialised torch.distributed group (any backend)")
        self.group = group
        self.nranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.nranks > _lib.MAX_PEERS:
            raise ValueError(f"at most {_lib.MAX_PEERS} expert-parallel ranks")
        self.device = device
        self.windows: list[Window] = []

    def window(self, nbytes: int) -> Window:
        w = Window(self, nbytes)
        self.windows.append(w)
        return w

    def free(self, windows) -> None:
        """Collective release of arena windows (every rank passes its windows in the same order)."""
        for w in windows:
            w.close()
            if w in self.windows:
                self.windows.remove(w)

    def close(self) -> None:
        self.free(list(self.windows))

    def measure_a2a(self, e_loc: int, c_i: int, width: int, dtype: torch.dtype, reps: int = 3) -> tuple[float, int]:
        """(seconds, elements received) of one dispatch-type chunk exchange of c_i rows per
        (source, local expert) on the current stream (calibration of w_comm; collective)."""
        esz = torch.empty((), dtype=dtype).element_size()
        N = self.nranks
        L = WindowLayout(N, N * e_loc, c_i, width, esz, 1, 4)
        win = Window(self, L.total)
        dst = torch.empty(e_loc * N * c_i * width, device=win._bytes.device, dtype=dtype)
        counter = torch.zeros(1, device=win._bytes.device, dtype=torch.int32)
        one = ctypes.c_uint32(1)
        ready = lower_plan(signal_plan(L, self.rank, FLAG_TI_READY), win.bases, {})
        pull = lower_plan(pull_plan(L, self.rank, e_loc, c_i, c_i, 0, "t_i", FLAG_TI_READY, ("loc", "x", 0),
                                    N * c_i, 0, reset=True), win.bases, {"x": dst.data_ptr()}, counter.data_ptr())
        stream = torch.cuda.current_stream()
        times = []
        for it in range(reps + 1):
            dist.barrier(group=self.group)  # every rank reset the previous repetition's flags
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _lib.call("mpm_p2p_run", ctypes.byref(ready), one, _s(stream))
            _lib.call("mpm_p2p_run", ctypes.byref(pull), one, _s(stream))
            b.record(stream)
            b.synchronize()
            if it:
                times.append(a.elapsed_time(b) * 1e-3)
        win.close()
        times.sort()
        return times[len(times) // 2], dst.numel()


def p2p_supported(group=None, device=None) -> bool:
    """Collective check that every rank can map every peer's IPC window (all GPUs visible to all
    ranks, peer access available); the answer is the same on every rank."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ptr = ctypes.c_void_p()
    handle = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
    ok = 1
    try:
        _lib.call("mpm_ipc_alloc", 4096, ctypes.byref(ptr), ctypes.cast(handle, ctypes.c_void_p))
    except _lib.MpmError:
        ok = 0
    handles = [None] * world
    dist.all_gather_object(handles, bytes(handle) if ok else None, group=group)
    opened = []
    for r, h in enumerate(handles):
        if r == rank or not ok:
            continue
        if h is None:
            ok = 0
            break
        p = ctypes.c_void_p()
        try:
            hb = (ctypes.c_char * _lib.IPC_HANDLE_BYTES).from_buffer_copy(h)
            _lib.call("mpm_ipc_open", ctypes.cast(hb, ctypes.c_void_p), ctypes.byref(p))
            opened.append(p.value)
        except _lib.MpmError:
            ok = 0
    flags = [None] * world
    dist.all_gather_object(flags, ok, group=group)
    for p in opened:
        _lib.call("mpm_ipc_close", ctypes.c_void_p(p))
    dist.barrier(group=group)
    if ptr.value:
        _lib.call("mpm_ipc_free", ptr)
    return all(bool(f) for f in flags)


def make_comm(backend: str, group=None, device=None):
    """The expert-parallel communicator for `backend` ("p2p" | "nccl"); single rank -> ExpertComm (identity).

    "p2p" (the product path) needs every peer's memory mappable from every rank (one process per GPU
    with every GPU of the node visible, as torchrun launches it).  When it is not, every rank raises:
    the exchanges never switch engines silently.  "nccl" is the explicitly chosen baseline."""
    if backend not in ("p2p", "nccl"):
        raise ValueError(f"a2a backend must be 'p2p' or 'nccl', got {backend!r}")
    if backend == "p2p" and dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if not p2p_supported(group, device):
            raise RuntimeError("a2a_backend='p2p': peer-memory windows cannot be mapped on every rank (each "
                               "process must see every GPU of the node; CUDA IPC and peer access required). "
                               "Pass a2a_backend='nccl' to run the NCCL send/recv baseline instead.")
        return PeerComm(group, device)
    return ExpertComm(group, device)


# ------------------------------------------------- p2p plans (symbolic)
# Addresses are symbolic until lowered: ("win", rank, byte offset) is a byte
# of rank's arena window, ("loc", name, byte offset) a byte of a local
# buffer.  The plans are plain integer arithmetic (CPU-testable: the gloo
# tests interpret them on numpy buffers); lower_plan turns one into the
# mpm_p2p_plan the C-ABI runs.
FLAG_TI_READY, FLAG_GO_READY, FLAG_DWG, FLAG_XS_FREE = 0, 1, 2, 3
FLAG_R0 = 4


def _align(v: int, a: int = 256) -> int:
    return (v + a - 1) // a * a


class WindowLayout:
    """Byte offsets inside every rank's arena window (identical on all ranks).

    t_i / t_o / g_o / g_i: the dispatch-side [E][C][M] buffers; with the
    fused dispatch (`fused`, no memory reuse) t_i / g_o are replaced by the
    expert-side t_di / g_do [E_loc][N*C][M] (same size) that peers push into;
    stage: the gate-gradient slices [N][E*M] f32; flags: uint32 [slots][N]
    with slots TI_READY, GO_READY, DWG, XS_FREE, R_i (n), BR_i (n), S_i (n),
    BS_i (n) — flag (slot, src) is raised (to 1) only by rank src and reset
    (to 0) only by the window's owner, after its last wait on it in the step.

    One stage buffer and one flag per exchange suffice across steps: a peer
    can raise a flag (or overwrite a stage slice) for step s+1 only after
    this rank has started step s+1 — every step begins with an all-to-all
    whose rows this rank provides only after its step s finished — and the
    resets / sums of step s are stream-ordered before that.
    """

    def __init__(self, N: int, E: int, C: int, M: int, esz: int, n: int, stage_elems: int,
                 fused: bool = False) -> None:
        self.N, self.n, self.fused = N, n, fused
        self.row_bytes = M * esz
        buf = E * C * M * esz
        off = 0
        self.off = {}
        for name in (("t_di", "t_o", "g_do", "g_i") if fused else ("t_i", "t_o", "g_o", "g_i")):
            self.off[name] = off
            off = _align(off + buf)
        self.stage_slice = _align(stage_elems * 4, 16)
        self.off["stage"] = off
        off = _align(off + N * self.stage_slice)
        self.off["kept"] = off  # [N][E] int32: every source's kept counts (compacted fused dispatch)
        self.kept_row = E * 4
        off = _align(off + N * E * 4)
        self.off["flags"] = off
        self.n_slots = FLAG_R0 + 4 * n
        self.total = _align(off + self.n_slots * N * 4)

    def flag(self, slot: int, src: int) -> int:
        return self.off["flags"] + (slot * self.N + src) * 4

    def r_slot(self, i: int) -> int:
        return FLAG_R0 + i

    def br_slot(self, i: int) -> int:
        return FLAG_R0 + self.n + i

    def s_slot(self, i: int) -> int:
        return FLAG_R0 + 2 * self.n + i

    def bs_slot(self, i: int) -> int:
        return FLAG_R0 + 3 * self.n + i

    def stage(self, rank: int) -> int:
        return self.off["stage"] + rank * self.stage_slice


def pull_plan(L: WindowLayout, rank: int, e_loc: int, C: int, c_i: int, s_i: int, src: str, ready_slot: int | None,
              dst, x_stride: int, x_row0: int, reset: bool = False, e0: int = 0, ne: int | None = None) -> dict:
    """Dispatch-type exchange at receiver `rank`: wait for every source's ready flag, then
    copy its [E_loc][c_i] rows addressed to this rank into the local expert rows
    (source p's rows of local expert el at el*x_stride + x_row0 + p*c_i; block_plan's layout).
    ready_slot None: no wait (a re-dispatch reads rows an earlier pull of the step already
    waited for); reset: this is the step's last wait on the ready flags, reset them after.
    The chunk covers local experts [e0, e0+ne) (block_plan's expert-side rows)."""
    rb = L.row_bytes
    ne = e_loc - e0 if ne is None else ne
    kind, name, base = dst
    copies = []
    for p in range(L.N):
        copies.append(((kind, name, base + (x_row0 + p * c_i) * rb),
                       ("win", p, L.off[src] + ((rank * e_loc + e0) * C + s_i) * rb),
                       x_stride * rb, C * rb, c_i * rb, ne))
    waits = [] if ready_slot is None else [("win", rank, L.flag(ready_slot, p)) for p in range(L.N) if p != rank]
    return {"wait": waits, "copy": copies, "signal": [], "arrive": [], "reset": list(waits) if reset else []}


def push_plan(L: WindowLayout, rank: int, e_loc: int, C: int, c_i: int, s_i: int, dst: str, slot: int,
              src, x_stride: int, x_row0: int, e0: int = 0, ne: int | None = None) -> dict:
    """Combine-type exchange at expert rank `rank`: copy the rows of every owner d into d's
    window, raise (slot, rank) there, then wait until every peer's rows have landed here
    (and reset those arrival flags: this is their only wait of the step)."""
    rb = L.row_bytes
    ne = e_loc - e0 if ne is None else ne
    kind, name, base = src
    copies = []
    for d in range(L.N):
        copies.append((("win", d, L.off[dst] + ((rank * e_loc + e0) * C + s_i) * rb),
                       (kind, name, base + (x_row0 + d * c_i) * rb),
                       C * rb, x_stride * rb, c_i * rb, ne))
    arrive = [("win", rank, L.flag(slot, p)) for p in range(L.N) if p != rank]
    return {"wait": [], "copy": copies,
            "signal": [("win", d, L.flag(slot, rank)) for d in range(L.N) if d != rank],
            "arrive": arrive, "reset": list(arrive)}


def push_dispatch_plan(L: WindowLayout, rank: int, e_loc: int, C: int, c_i: int, s_i: int, dst: str, slot: int,
                       e0: int = 0, ne: int | None = None) -> dict:
    """Fused dispatch of one chunk at source `rank` (mpm_dispatch_push): every destination d's
    expert-side buffer `dst` (window) receives this rank's rows of local experts [e0, e0+ne), slots
    [s_i, s_i+c_i) at (el-e0)*N*C + e0*N*C + N*s_i + rank*c_i + (s - s_i) — block_plan's full-buffer
    layout — and flag (slot, rank) is raised in every peer's window; the op then waits for the
    peers' flags of this chunk in its own window and resets them."""
    ne = e_loc - e0 if ne is None else ne
    arrive = [("win", rank, L.flag(slot, p)) for p in range(L.N) if p != rank]
    return {"dst": [("win", d, L.off[dst]) for d in range(L.N)],
            "flag": [("win", d, L.flag(slot, rank)) for d in range(L.N)],
            "geom": dict(e_loc=e_loc, capacity=C, e0=e0, ne=ne, s0=s_i, cs=c_i, x_stride=L.N * C,
                         x_row0=e0 * L.N * C + L.N * s_i),
            "arrive": arrive, "reset": list(arrive)}


def kept_signal_plan(L: WindowLayout, rank: int, slot: int = FLAG_XS_FREE) -> dict:
    """A once-per-step signal of the compacted layout that carries this rank's kept[E]: copy it into
    every rank's window row `rank` of the kept table, then raise (slot, rank) in every peer.  XS_FREE
    (fused dispatch: S_0 waits for it, so a sender holds every source's counts — the row offsets — before
    it pushes) or TI_READY (memory reuse: every pull waits for it before reading the sources' rows)."""
    off = L.off["kept"] + rank * L.kept_row
    return {"wait": [], "copy": [(("win", d, off), ("loc", "kept", 0), L.kept_row, L.kept_row, L.kept_row, 1)
                                 for d in range(L.N)],
            "signal": [("win", d, L.flag(slot, rank)) for d in range(L.N) if d != rank],
            "arrive": [], "reset": []}


def compact_pull_plan(L: WindowLayout, rank: int, e_loc: int, C: int, c_i: int, s_i: int, src: str,
                      x_stride: int, x_row0: int, e0: int = 0, ne: int | None = None) -> dict:
    """Dispatch-type pull of one chunk into the compacted layout (mpm_compact_pull): every source s's
    dispatch-side buffer `src` (window) is read; the ready-flag waits / resets stay in mpm_p2p_run."""
    ne = e_loc - e0 if ne is None else ne
    return {"dst": [("win", s_, L.off[src]) for s_ in range(L.N)], "flag": [],
            "geom": dict(e_loc=e_loc, capacity=C, e0=e0, ne=ne, s0=s_i, cs=c_i, x_stride=x_stride, x_row0=x_row0)}


def combine_push_plan(L: WindowLayout, rank: int, e_loc: int, C: int, c_i: int, s_i: int, dst: str, slot: int,
                      x_stride: int, x_row0: int, e0: int = 0, ne: int | None = None) -> dict:
    """Combine-type exchange in the compacted layout (mpm_combine_push): every owner d's routed rows of
    this rank's experts [e0, e0+ne) go to d's dispatch-side buffer `dst`, flag (slot, rank) is raised
    in every peer, then the op waits for (and resets) the peers' flags in its own window."""
    ne = e_loc - e0 if ne is None else ne
    arrive = [("win", rank, L.flag(slot, p)) for p in range(L.N) if p != rank]
    return {"dst": [("win", d, L.off[dst]) for d in range(L.N)],
            "flag": [("win", d, L.flag(slot, rank)) for d in range(L.N)],
            "geom": dict(e_loc=e_loc, capacity=C, e0=e0, ne=ne, s0=s_i, cs=c_i, x_stride=x_stride, x_row0=x_row0),
            "arrive": arrive, "reset": list(arrive)}


def lower_push(plan: dict, win_bases: list[int], rank: int, counter: int) -> "_lib.PushPlan":
    out = _lib.PushPlan()
    out.nranks, out.rank = len(plan["dst"]), rank
    for d, (_, r, off) in enumerate(plan["dst"]):
        out.dst[d] = win_bases[r] + off
    for d, (_, r, off) in enumerate(plan.get("flag", [])):
        out.flag[d] = win_bases[r] + off
    for k_, v in plan["geom"].items():
        setattr(out, k_, v)
    out.counter = counter
    if plan.get("kept_all") is not None:  # compacted layout: this rank's copy of every source's counts
        _, r, off = plan["kept_all"]
        out.kept_all = win_bases[r] + off
    return out


def signal_plan(L: WindowLayout, rank: int, slot: int) -> dict:
    """Raise (slot, rank) in every peer's window (e.g. "my T_I is ready to be pulled")."""
    return {"wait": [], "copy": [], "signal": [("win", d, L.flag(slot, rank)) for d in range(L.N) if d != rank],
            "arrive": [], "reset": []}


def reduce_plan(L: WindowLayout, rank: int, nbytes: int) -> dict:
    """Gate-gradient all-reduce, step 1: push this rank's slice into every peer's
    stage[rank], then wait for all slices (mpm_sum_slices adds them in rank order)."""
    off = L.stage(rank)
    arrive = [("win", rank, L.flag(FLAG_DWG, p)) for p in range(L.N) if p != rank]
    return {"wait": [], "copy": [(("win", d, off), ("win", rank, off), nbytes, nbytes, nbytes, 1)
                                 for d in range(L.N) if d != rank],
            "signal": [("win", d, L.flag(FLAG_DWG, rank)) for d in range(L.N) if d != rank],
            "arrive": arrive, "reset": list(arrive)}


def lower_plan(plan: dict, win_bases: list[int], locals_: dict, counter: int = 0) -> "_lib.P2PPlan":
    """Symbolic plan -> mpm_p2p_plan (device addresses); `counter` is the plan's own zeroed
    device uint32 for the SM copy kernel's completion count (needed when the plan copies)."""
    def addr(sym) -> int:
        kind, key, off = sym
        return (win_bases[key] if kind == "win" else locals_[key]) + off

    out = _lib.P2PPlan()
    out.n_wait = len(plan["wait"])
    for j, w in enumerate(plan["wait"]):
        out.wait[j] = addr(w)
    out.n_copy = len(plan["copy"])
    for j, (dst, src, dp, sp, width, height) in enumerate(plan["copy"]):
        c = out.copy[j]
        c.dst, c.src, c.dpitch, c.spitch, c.width, c.height = addr(dst), addr(src), dp, sp, width, height
    out.n_signal = len(plan["signal"])
    for j, sgl in enumerate(plan["signal"]):
        out.signal[j] = addr(sgl)
    out.n_arrive = len(plan["arrive"])
    for j, a in enumerate(plan["arrive"]):
        out.arrive[j] = addr(a)
    out.n_reset = len(plan.get("reset", []))
    for j, r in enumerate(plan.get("reset", [])):
        out.reset[j] = addr(r)
    out.counter = counter or None
    return out
