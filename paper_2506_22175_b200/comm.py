"""Expert-parallel communicator: an NCCL comm owned by libmpm (C-ABI).

The unique id is created by rank 0 through mpm_comm_unique_id and broadcast
with torch.distributed (any backend), then every rank calls mpm_comm_init.
With one rank (or no process group) no NCCL communicator is created: the
chunk all-to-alls degenerate to identities (PAPER.md:520 / SURVEY.md §8e).
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .ops import _p, _s, dtype_code


def block_plan(direction: int, nranks: int, e_loc: int, c_i: int, width: int, capacity: int, s_i: int,
               x_stride: int, x_row0: int) -> tuple[list[int], list[int], list[int]]:
    """(peer, send offset, recv offset) in elements per block of c_i*width elements.

    Source side (dispatch): this rank's expert-major buffer [E][C][W]; the
    block for (peer d, local expert el) is rows [(d*E_loc+el)*C + s_i, +c_i).
    Expert side: local expert el's region starts at row el*x_stride and the
    chunk's rows start at x_row0, source-major (source s at + s*c_i).  A
    full (all-chunk) buffer uses x_stride = N*C, x_row0 = N*s_i; a per-chunk
    ring slot x_stride = N*c_i, x_row0 = 0.  Combine is the inverse.  Blocks
    are ordered (peer, el) on every rank, so the b-th send to a peer pairs
    with that peer's b-th receive from this rank.
    """
    peers, send, recv = [], [], []
    for peer in range(nranks):
        for el in range(e_loc):
            source = ((peer * e_loc + el) * capacity + s_i) * width
            expert = (el * x_stride + x_row0 + peer * c_i) * width
            peers.append(peer)
            if direction == _lib.A2A_DISPATCH:
                send.append(source)
                recv.append(expert)
            else:
                send.append(expert)
                recv.append(source)
    return peers, send, recv


class ExpertComm:
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
