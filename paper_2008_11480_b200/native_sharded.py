"""Block-row sharded steps through the C ABI (``si_comm_*`` / ``si_sharded_*``).

The multi-GPU path of :mod:`sharded` with its orchestration in the native
library: one call per step, the library computes this rank's rows of every
product of the reference DAG and all-gathers the sharded right operands
itself (NCCL, or a caller-provided exchange).  A C / cgo / JNI host gets the
same path through ``include/seriesinv_b200.h``; this module is the Python
mirror (same names and arguments as the single-GPU steps, row blocks in and
out), SURVEY 8(b) / 8(e).

Communicators:

* :meth:`NativeComm.nccl` -- NCCL (one rank per GPU; the unique id is
  broadcast over the ``torch.distributed`` group).
* :meth:`NativeComm.host` -- the exchange runs through ``torch.distributed``
  on host copies (gloo): slow, but lets several processes share one GPU in
  tests (no kernel ever waits on another process).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .matrix_core import MulCounter, as_device
from .series_toolkit import FactorPlan, encode_many, encode_plan, geometric_base_plan

__all__ = ["NativeComm", "composite_step", "fro_norm", "ns_step", "plain_richardson",
           "richardson_recursive_step"]

_AG = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_int64, ctypes.c_void_p)
_AR = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                       ctypes.c_void_p)


class NativeComm:
    """An ``si_comm``: the row split of n over the group and its exchange."""

    def __init__(self, ptr: int, n: int, rank: int, world: int, device: torch.device,
                 keep=None):
        self.ptr, self.n, self.rank, self.world, self.device = ptr, n, rank, world, device
        self._keep = keep  # callback objects must outlive the communicator
        r0, r1 = ctypes.c_int64(), ctypes.c_int64()
        _lib.call("si_comm_rows", ptr, ctypes.byref(r0), ctypes.byref(r1), None, None)
        self.r0, self.r1 = r0.value, r1.value

    @classmethod
    def nccl(cls, n: int, group=None) -> "NativeComm":
        import torch.distributed as dist

        dev = torch.device("cuda", torch.cuda.current_device())
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        uid = (ctypes.c_ubyte * 128)()
        if rank == 0:
            _lib.call("si_comm_unique_id", uid)
        if world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                                       group=group)
            uid = (ctypes.c_ubyte * 128).from_buffer_copy(box[0])
        out = ctypes.c_void_p()
        _lib.call("si_comm_create_nccl", _lib.handle(dev.index), world, rank, uid, n,
                  ctypes.byref(out))
        return cls(out.value, n, rank, world, dev)

    @classmethod
    def host(cls, n: int, group=None) -> "NativeComm":
        """Exchange over torch.distributed on host copies (tests / 1-GPU boxes)."""
        import torch.distributed as dist

        dev = torch.device("cuda", torch.cuda.current_device())
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        h = _lib.handle(dev.index)

        def to_host(ptr, count, stream):
            t = torch.empty(count, dtype=torch.float64, pin_memory=True)
            _lib.call("si_copy_async", h, t.data_ptr(), ptr, count * 8, stream)
            torch.cuda.current_stream(dev).synchronize()
            torch.cuda.synchronize(dev)
            return t

        def allgather(_ctx, send, recv, count, stream):
            try:
                mine = to_host(send, count, stream)
                parts = [torch.empty(count, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, mine, group=group)
                host = torch.cat(parts).pin_memory()
                _lib.call("si_copy_async", h, recv, host.data_ptr(), world * count * 8, stream)
                torch.cuda.synchronize(dev)
                return 0
            except Exception:  # noqa: BLE001 -- reported as a failed exchange
                return 1

        def allreduce(_ctx, buf, count, stream):
            try:
                t = to_host(buf, count, stream).clone()
                dist.all_reduce(t, group=group)
                host = t.pin_memory()
                _lib.call("si_copy_async", h, buf, host.data_ptr(), count * 8, stream)
                torch.cuda.synchronize(dev)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        ag, ar = _AG(allgather), _AR(allreduce)
        out = ctypes.c_void_p()
        _lib.call("si_comm_create_callback", world, rank, n, ag, ar, None, ctypes.byref(out))
        return cls(out.value, n, rank, world, dev, keep=(ag, ar))

    def stats(self) -> tuple[int, int]:
        """(all-gathers so far, bytes received from the other ranks)."""
        g, b = ctypes.c_int64(), ctypes.c_int64()
        _lib.call("si_comm_rows", self.ptr, None, None, ctypes.byref(g), ctypes.byref(b))
        return g.value, b.value

    def close(self):
        if self.ptr:
            _lib.call("si_comm_destroy", self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass

    def rows_of(self, full: torch.Tensor) -> torch.Tensor:
        return full[self.r0:self.r1].contiguous()


def _rows(comm: NativeComm, x) -> torch.Tensor:
    x = as_device(x).contiguous()
    if x.shape[0] != comm.r1 - comm.r0 or x.shape[1] != comm.n:
        raise ValueError("row block does not match this rank's split")
    return x


def _ctx(comm: NativeComm):
    return _lib.handle(comm.device.index), _lib.stream_ptr(comm.device)


def ns_step(comm: NativeComm, g_rows, f_rows, a, order: int, plan: FactorPlan | None = None,
            ctr: MulCounter | None = None):
    """newton_schulz.py:150-174 on row blocks; returns (G' rows, F' rows)."""
    g_rows, f_rows, a = _rows(comm, g_rows), _rows(comm, f_rows), as_device(a)
    code, consts = encode_plan(plan) if plan is not None else ([], [])
    g, f = torch.empty_like(g_rows), torch.empty_like(f_rows)
    h, s = _ctx(comm)
    buf = _lib.counter_buf()
    _lib.call("si_sharded_ns_step", h, comm.ptr, comm.n, a.data_ptr(), g_rows.data_ptr(),
              f_rows.data_ptr(), order, _lib.i32_array(code) if code else None, len(code),
              _lib.f64_array(consts) if consts else None, len(consts), g.data_ptr(), f.data_ptr(),
              buf, s)
    if ctr is not None:
        ctr.absorb(buf)
    return g, f


def composite_step(comm: NativeComm, g_rows, f_rows, a, precond, residual, split_matrix, rates,
                   order_n: int, ctr: MulCounter | None = None):
    """newton_schulz.py:177-228 on row blocks; returns (G' rows, F' rows)."""
    g_rows, f_rows = _rows(comm, g_rows), _rows(comm, f_rows)
    a, precond, residual, split_matrix = (as_device(x) for x in (a, precond, residual, split_matrix))
    rates = tuple(int(x) for x in rates)
    plans = [geometric_base_plan(x) if x > 1 else None for x in rates]
    code, offsets, consts = encode_many(plans)
    g, f = torch.empty_like(g_rows), torch.empty_like(f_rows)
    h, s = _ctx(comm)
    buf = _lib.counter_buf()
    _lib.call("si_sharded_composite_step", h, comm.ptr, comm.n, a.data_ptr(), g_rows.data_ptr(),
              f_rows.data_ptr(), precond.data_ptr(), residual.data_ptr(), split_matrix.data_ptr(),
              len(rates), _lib.i32_array(list(rates)), _lib.i32_array(code),
              _lib.i64_array(offsets), _lib.f64_array(consts), len(consts), order_n, g.data_ptr(),
              f.data_ptr(), buf, s)
    if ctr is not None:
        ctr.absorb(buf)
    return g, f


def plain_richardson(comm: NativeComm, theta, p_rows, a, b, ctr: MulCounter | None = None):
    """theta - P (A theta - b) with P row-sharded; theta replicated in and out."""
    theta, a, b = as_device(theta).contiguous(), as_device(a), as_device(b).contiguous()
    p_rows = _rows(comm, p_rows)
    r = theta.shape[1] if theta.ndim == 2 else 1
    out = torch.empty_like(theta)
    h, s = _ctx(comm)
    buf = _lib.counter_buf()
    _lib.call("si_sharded_plain_richardson", h, comm.ptr, comm.n, r, a.data_ptr(), b.data_ptr(),
              theta.data_ptr(), p_rows.data_ptr(), out.data_ptr(), buf, s)
    if ctr is not None:
        ctr.absorb(buf)
    return out


def richardson_recursive_step(comm: NativeComm, state: list, a, theta, b, order: int,
                              factor_plan: FactorPlan | None = None, doubling_sum: bool = False,
                              ctr: MulCounter | None = None):
    """richardson.py:111-189 on row blocks.  ``state`` = [G, F, L, R, omega, N]
    row blocks (omega / N None on the first call); returns (new state, theta')."""
    g, f, l, r, om, ns = state
    g, f, l, r = (_rows(comm, x) for x in (g, f, l, r))
    if (om is None) != (ns is None):
        raise ValueError("omega and ns_part go together")
    if om is not None:
        om, ns = _rows(comm, om), _rows(comm, ns)
    theta, a, b = as_device(theta).contiguous(), as_device(a), as_device(b).contiguous()
    nrhs = theta.shape[1] if theta.ndim == 2 else 1
    code, consts = encode_plan(factor_plan) if factor_plan is not None else ([], [])
    outs = [torch.empty_like(g) for _ in range(6)]
    th = torch.empty_like(theta)
    h, s = _ctx(comm)
    buf = _lib.counter_buf()
    _lib.call("si_sharded_richardson_recursive_step", h, comm.ptr, comm.n, nrhs, a.data_ptr(),
              b.data_ptr(), theta.data_ptr(), g.data_ptr(), f.data_ptr(), l.data_ptr(),
              r.data_ptr(), om.data_ptr() if om is not None else None,
              ns.data_ptr() if ns is not None else None, order,
              _lib.i32_array(code) if code else None, len(code),
              _lib.f64_array(consts) if consts else None, len(consts), int(doubling_sum),
              *[o.data_ptr() for o in outs], th.data_ptr(), buf, s)
    if ctr is not None:
        ctr.absorb(buf)
    return outs, th


def fro_norm(comm: NativeComm, x_rows) -> float:
    """||X||_F of a row-sharded matrix (local sums + one all-reduce)."""
    x_rows = as_device(x_rows).contiguous()
    out = ctypes.c_double()
    h, s = _ctx(comm)
    _lib.call("si_sharded_fro_norm", h, comm.ptr, comm.n, x_rows.shape[1], x_rows.data_ptr(),
              ctypes.byref(out), s)
    return out.value
