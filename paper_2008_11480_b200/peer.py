"""Row-panel exchange over peer memory for the block-row sharded path.

The one exchange step of the sharded hot path is the all-gather of a
row-sharded right operand before ``L[rows] @ R`` (every ``mat_mul(y, x)``
with ``x`` sharded, matrix_core.py:101-106).  :class:`PeerComm` does it without
NCCL and without SMs:

* every rank owns one exchange buffer per live gathered value ("slot", the
  full n x c matrix), allocated with ``cudaMalloc`` and mapped into every peer
  process through CUDA IPC (``si_sym_alloc`` / ``si_sym_open``);
* the producer copies its row block into its own slot and raises a
  ``published`` flag in every peer's flag array (stream memory operation,
  ordered after the copy);
* each peer pulls the block with a copy engine (``cudaMemcpyAsync`` from the
  IPC mapping, over NVLink) on its copy stream, which first waits for the
  flag, then raises its local ``ready`` flag for that panel and the owner's
  ``consumed`` flag (slot reuse waits for it);
* the consuming product either gates its TMA loads panel by panel on the
  ``ready`` flags inside the DMMA kernel (``si_gemm_panels``, mode "fused":
  the gather overlaps the product k-slab by k-slab) or, mode "stream", the
  compute stream waits for the copies before the launch.

Copy engines matter on B200: the DMMA GEMM is a persistent kernel holding
every SM (one 200 KB CTA each), so an SM-driven collective queued beside it
cannot run until it finishes, while copy engines and stream memory operations
need no SM.

The same class runs P "virtual ranks" in one process on one GPU
(:class:`LocalFabric`, used by the GPU tests): buffers are plain allocations
and peers are the other virtual ranks.  Virtual ranks must use mode "stream"
(a spinning kernel of one virtual rank could hold the SMs another virtual
rank's producer needs); the fused gate is tested at kernel level.

Streams that wait on flags must not share a hardware work queue with a stream
that has to make progress meanwhile: processes using this module set
``CUDA_DEVICE_MAX_CONNECTIONS`` (32) before CUDA starts (bench.py, the tests),
and each rank uses two streams (compute + copy).
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from .sharded import row_splits

__all__ = ["GatedOperand", "IpcFabric", "LocalFabric", "PeerComm"]

_MAX_PANELS = 16        # kMaxPanels in csrc/common.cuh
_MAX_SLOTS = 256
_FLAG_WORDS = 3 * _MAX_SLOTS * _MAX_PANELS   # published / ready / consumed


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory.  The tensor built
    from it keeps this object (and its ``lease``) alive."""

    def __init__(self, ptr: int, shape, lease=None):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": "<f8", "data": (ptr, False),
            "version": 3, "strides": None, "stream": None}
        self.lease = lease


def _tensor(ptr: int, shape, device, lease=None) -> torch.Tensor:
    return torch.as_tensor(_CudaArray(ptr, shape, lease), device=device)


class IpcFabric:
    """Exchange buffers shared between the ranks of a torch.distributed group
    (one process per GPU) through CUDA IPC handles."""

    def __init__(self, device: torch.device, group=None):
        import torch.distributed as dist

        self.dist, self.group, self.device = dist, group, device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._owned, self._opened = [], []

    def alloc(self, nbytes: int) -> tuple[int, list[int]]:
        """Collective: every rank allocates ``nbytes``; returns (own pointer,
        pointers of all ranks' buffers as mapped here)."""
        h = _lib.handle(self.device.index)
        ptr = ctypes.c_void_p()
        raw = (ctypes.c_ubyte * 64)()
        _lib.call("si_sym_alloc", h, nbytes, ctypes.byref(ptr), raw)
        self._owned.append(ptr.value)
        handles = [None] * self.world
        self.dist.all_gather_object(handles, bytes(raw), group=self.group)
        ptrs = []
        for r, hb in enumerate(handles):
            if r == self.rank:
                ptrs.append(ptr.value)
                continue
            peer = ctypes.c_void_p()
            _lib.call("si_sym_open", h, (ctypes.c_ubyte * 64)(*hb), ctypes.byref(peer))
            self._opened.append(peer.value)
            ptrs.append(peer.value)
        return ptr.value, ptrs

    def close(self):
        h = _lib.handle(self.device.index)
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            self.dist.barrier(group=self.group)  # no peer still reads our buffers
        for p in self._opened:
            _lib.call("si_sym_close", h, p)
        for p in self._owned:
            _lib.call("si_sym_free", h, p)
        self._owned, self._opened = [], []


class LocalFabric:
    """P virtual ranks in one process on one GPU: ``alloc`` call number i of
    every virtual rank returns the i-th group of P buffers (SPMD order).

    Buffers are allocated and zeroed on the fabric's own stream and completed
    before they are handed out: a virtual rank's stream may be blocked on a
    flag another virtual rank has not raised yet, so nothing of the fabric may
    be queued behind it."""

    def __init__(self, device: torch.device, world: int):
        self.device, self.world = device, world
        self._groups: list[list[torch.Tensor]] = []
        self._calls = [0] * world
        self._stream = torch.cuda.Stream(device=device)

    def view(self, rank: int) -> "_LocalView":
        return _LocalView(self, rank)

    def _alloc(self, rank: int, nbytes: int) -> tuple[int, list[int]]:
        i = self._calls[rank]
        self._calls[rank] += 1
        if i == len(self._groups):
            words = (nbytes + 7) // 8
            with torch.cuda.stream(self._stream):
                grp = [torch.zeros(words, dtype=torch.float64, device=self.device)
                       for _ in range(self.world)]
            self._stream.synchronize()
            self._groups.append(grp)
        grp = self._groups[i]
        return grp[rank].data_ptr(), [t.data_ptr() for t in grp]


class _LocalView:
    def __init__(self, fabric: LocalFabric, rank: int):
        self.fabric, self.rank, self.world, self.device = fabric, rank, fabric.world, fabric.device

    def alloc(self, nbytes: int):
        return self.fabric._alloc(self.rank, nbytes)

    def close(self):
        pass


class _Slot:
    __slots__ = ("index", "shape", "ptr", "peers", "epoch", "busy", "reserved")

    def __init__(self, index, shape, ptr, peers):
        self.index, self.shape, self.ptr, self.peers = index, shape, ptr, peers
        self.epoch = 0
        self.busy = False
        self.reserved = 0  # epoch handed to an in-place producer (output_rows)


class _Lease:
    """Keeps a slot reserved while anything (pending exchange, gated operand,
    tensor view) may still read it."""

    def __init__(self, slot: _Slot):
        self.slot = slot
        slot.busy = True

    def __del__(self):
        self.slot.busy = False


class GatedOperand:
    """A gathered right operand whose row panels may still be in flight:
    ``t`` is the full matrix, panel p (rows ``bounds[p]:bounds[p+1]``) is valid
    once ``*(ready + 4 p) >= epoch``."""

    def __init__(self, t: torch.Tensor, ready: int, epoch: int, bounds: list[int], lease):
        self.t, self.ready, self.epoch, self.bounds, self.lease = t, ready, epoch, bounds, lease
        self.shape = t.shape


class _Pending:
    __slots__ = ("slot", "keep", "epoch", "events", "rows", "cols")

    def __init__(self, slot, keep, epoch, events, rows, cols):
        # `keep` holds the slot's lease (directly, or through the producer's
        # in-place output view) while the exchange may still read it
        self.slot, self.keep, self.epoch, self.events = slot, keep, epoch, events
        self.rows, self.cols = rows, cols


class PeerComm:
    """Drop-in for :class:`~paper_2008_11480_b200.sharded.RowComm` (same
    ``start_gather`` / ``finish`` interface) that moves row panels over peer
    memory; ``gate`` returns a :class:`GatedOperand` for fused products."""

    def __init__(self, n: int, fabric, mode: str = "fused"):
        if mode not in ("fused", "stream"):
            raise ValueError("mode must be 'fused' or 'stream'")
        self.fabric = fabric
        self.rank, self.world, self.device = fabric.rank, fabric.world, fabric.device
        if self.world > _MAX_PANELS:
            raise ValueError(f"at most {_MAX_PANELS} ranks")
        self.mode = mode
        self.n = n
        self.splits = row_splits(n, self.world)
        self.r0, self.r1 = self.splits[self.rank]
        self.bounds = [s[0] for s in self.splits] + [n]
        self.bytes_gathered = 0
        self.local_copies = 0  # row blocks copied into a slot (not produced in place)
        # gathers started so far; with SI_PEER_CHECK=1 every start_gather
        # all-gathers (seq, slot, epoch, cols) over the group and raises if the
        # ranks paired different slots (slot choice follows lease lifetimes, so
        # a rank-dependent branch or a held reference could desynchronise them:
        # the result would be wrong data, not a hang)
        self.seq = 0
        self._check = os.environ.get("SI_PEER_CHECK") == "1"
        self._slots: list[_Slot] = []
        self._cs = None
        self._h = _lib.handle(self.device.index)
        if self.world > 1:
            # zeroed (and completed) by the fabric before it returns
            self._flags, self._peer_flags = fabric.alloc(_FLAG_WORDS * 4)

    # -- flags: [kind][slot][rank] u32 --------------------------------------
    @staticmethod
    def _off(kind: int, slot: int, r: int) -> int:
        return 4 * ((kind * _MAX_SLOTS + slot) * _MAX_PANELS + r)

    def _flag(self, base: int, kind: int, slot: int, r: int) -> int:
        return base + self._off(kind, slot, r)

    _PUB, _READY, _CONSUMED = 0, 1, 2

    def _copy_stream(self) -> torch.cuda.Stream:
        if self._cs is None:
            self._cs = torch.cuda.Stream(device=self.device)
        return self._cs

    def _acquire(self, shape) -> _Slot:
        for s in self._slots:
            if not s.busy and s.shape == shape:
                s.reserved = 0  # an in-place reservation whose value died unpublished
                return s
        if len(self._slots) >= _MAX_SLOTS:
            raise MemoryError("too many live exchange slots")
        nbytes = shape[0] * shape[1] * 8
        ptr, peers = self.fabric.alloc(nbytes)
        s = _Slot(len(self._slots), shape, ptr, peers)
        self._slots.append(s)
        return s

    # -- RowComm interface ---------------------------------------------------
    def all_gather_rows(self, local: torch.Tensor) -> torch.Tensor:
        return self.finish(self.start_gather(local))

    def _war_wait(self, slot: _Slot, e: int, stream_ptr: int) -> None:
        """Peers have finished pulling our previous block out of this slot."""
        if e > 1:
            for q in range(self.world):
                if q != self.rank:
                    _lib.call("si_stream_wait_u32", self._h,
                              self._flag(self._flags, self._CONSUMED, slot.index, q), e - 1,
                              stream_ptr)

    def output_rows(self, cols: int):
        """This rank's row block inside a fresh exchange slot: a product written
        there is published by :meth:`start_gather` without a copy (the slot's
        reuse guard is queued now, before the producer writes)."""
        if self.world == 1:
            return None
        slot = self._acquire((self.n, cols))
        lease = _Lease(slot)
        e = slot.epoch + 1
        self._war_wait(slot, e, torch.cuda.current_stream(self.device).cuda_stream)
        slot.reserved = e
        return _tensor(slot.ptr + self.r0 * cols * 8, (self.r1 - self.r0, cols), self.device,
                       lease)

    def start_gather(self, local: torch.Tensor):
        """Publish this rank's row block and queue the pulls of the others'."""
        if self.world == 1:
            return (None, local)
        if local.shape[0] != self.r1 - self.r0:
            raise ValueError("row block does not match this rank's split")
        cols = local.shape[1]
        row_bytes = cols * 8
        h, me = self._h, self.rank
        cur = torch.cuda.current_stream(self.device)
        sp = cur.cuda_stream
        slot = next((sl for sl in self._slots if sl.reserved and sl.shape == (self.n, cols)
                     and sl.ptr + self.r0 * row_bytes == local.data_ptr()), None)
        if slot is not None:  # produced in place by output_rows: no copy
            keep = local
            slot.epoch, slot.reserved = slot.reserved, 0
            e, b = slot.epoch, slot.index
        else:
            slot = self._acquire((self.n, cols))
            keep = _Lease(slot)
            slot.epoch += 1
            e, b = slot.epoch, slot.index
            self._war_wait(slot, e, sp)
        if keep is not local:
            self.local_copies += 1
            src = local.contiguous()
            _lib.call("si_copy_async", h, slot.ptr + self.r0 * row_bytes, src.data_ptr(),
                      (self.r1 - self.r0) * row_bytes, sp)
        self.seq += 1
        if self._check:
            self._check_agreement(b, e, cols)
        for q in range(self.world):
            if q != me:
                _lib.call("si_stream_write_u32", h,
                          self._flag(self._peer_flags[q], self._PUB, b, me), e, sp)
        _lib.call("si_stream_write_u32", h, self._flag(self._flags, self._READY, b, me), e, sp)
        produced = torch.cuda.Event()
        produced.record(cur)
        # one copy stream, peers in ring order from the next rank: pulls of a
        # gather only wait for publications earlier in every rank's program
        # order, so the queue cannot deadlock (one stream also keeps the number
        # of streams within the device's hardware queues: a waiting stream
        # would block any stream sharing its queue)
        cs = self._copy_stream()
        cs.wait_event(produced)   # local readers of the previous epoch are done
        csp = cs.cuda_stream
        for i in range(1, self.world):
            q = (me + i) % self.world
            q0, q1 = self.splits[q]
            _lib.call("si_stream_wait_u32", h, self._flag(self._flags, self._PUB, b, q), e, csp)
            _lib.call("si_copy_async", h, slot.ptr + q0 * row_bytes,
                      slot.peers[q] + q0 * row_bytes, (q1 - q0) * row_bytes, csp)
            _lib.call("si_stream_write_u32", h, self._flag(self._flags, self._READY, b, q), e, csp)
            _lib.call("si_stream_write_u32", h,
                      self._flag(self._peer_flags[q], self._CONSUMED, b, me), e, csp)
        done = torch.cuda.Event()
        done.record(cs)
        events = [done]
        self.bytes_gathered += (self.n - (self.r1 - self.r0)) * row_bytes
        return _Pending(slot, keep, e, events, self.n, cols)

    def _check_agreement(self, slot: int, epoch: int, cols: int) -> None:
        """Debug mode (SI_PEER_CHECK=1): every rank must pair this gather with
        the same (slot, epoch); a divergence fails loudly instead of pulling
        another value's panels."""
        mine = (self.seq, slot, epoch, cols)
        if isinstance(self.fabric, IpcFabric):
            seen = [None] * self.world
            self.fabric.dist.all_gather_object(seen, mine, group=self.fabric.group)
        else:  # virtual ranks of one process: compare through the shared fabric
            shared = getattr(self.fabric, "fabric", self.fabric)  # _LocalView -> LocalFabric
            log = shared.__dict__.setdefault("_gather_log", {})
            seen = [log.setdefault(self.seq, mine)]
        if any(tuple(x) != mine for x in seen):
            raise RuntimeError(f"peer exchange diverged at gather {self.seq}: rank {self.rank} "
                               f"has (seq, slot, epoch, cols) = {mine}, the group {seen}")

    def _view(self, pend: _Pending) -> torch.Tensor:
        return _tensor(pend.slot.ptr, (pend.rows, pend.cols), self.device, pend.keep)

    def finish(self, pending) -> torch.Tensor:
        """The full matrix, with the current stream ordered after every pull."""
        if isinstance(pending, tuple):
            return pending[1]
        cur = torch.cuda.current_stream(self.device)
        for ev in pending.events:
            cur.wait_event(ev)
        return self._view(pending)

    def gate(self, pending):
        """A :class:`GatedOperand` (mode "fused") or the finished matrix."""
        if isinstance(pending, tuple) or self.mode != "fused":
            return self.finish(pending)
        ready = self._flag(self._flags, self._READY, pending.slot.index, 0)
        return GatedOperand(self._view(pending), ready, pending.epoch, list(self.bounds),
                            pending.keep)

    def barrier(self):
        if self.world > 1 and isinstance(self.fabric, IpcFabric):
            self.fabric.dist.barrier(group=self.fabric.group)

    def all_reduce_sum(self, x: float) -> float:
        """Scalar sum over the ranks (stop rule); host collective of the group."""
        if self.world == 1:
            return x
        if not isinstance(self.fabric, IpcFabric):
            raise NotImplementedError("scalar reductions need a process group (IpcFabric)")
        t = torch.tensor([x], dtype=torch.float64)
        self.fabric.dist.all_reduce(t, group=self.fabric.group)
        return float(t.item())

    def close(self):
        self.fabric.close()
