"""Batched small systems (BASELINE config 2) on the device.

``batched_composite_richardson`` advances ``batch`` independent n x n systems
(n <= 32) through ``iters`` x { plain Richardson with P_k;
``composite_step(rates, order_n)`` (newton_schulz.py:177-228) } in ONE kernel
launch: one CTA per system, the whole state resident in shared memory, DMMA
products.  Per system it executes exactly the reference GEMM DAG, so the
returned counter is the per-system MulCounter delta.
"""

from __future__ import annotations

import torch

from . import _lib
from .matrix_core import MulCounter, as_device
from .series_toolkit import encode_many, geometric_base_plan

__all__ = ["batched_composite_richardson", "batched_ns_richardson", "batched_scalar_split"]


def batched_scalar_split(a: torch.Tensor, eps_factor: float = 0.5):
    """Per-system split_scalar(A_i, eps = eps_factor*||A_i||_inf) (splitting.py:124-146):
    alpha_i = ||A_i||_inf (1/2 + eps_factor); P_i = I/alpha_i, B_i = I - A_i/alpha_i.
    ``eps_factor=0.5`` gives P0 = I/||A||_inf."""
    a = as_device(a)
    n = a.shape[-1]
    norm = a.abs().sum(dim=-1).amax(dim=-1)
    alpha = norm / 2.0 + eps_factor * norm
    eye = torch.eye(n, dtype=torch.float64, device=a.device)
    precond = eye / alpha[:, None, None]
    residual = eye - a / alpha[:, None, None]
    return precond, residual


def batched_composite_richardson(a, b, precond, residual, p, f, theta, rates, order_n: int,
                                 iters: int, ctr: MulCounter | None = None, *,
                                 input_chunks: tuple | None = None, chunk_done=None):
    """Returns new (P, F, theta) after ``iters`` fused iterations; inputs untouched.

    ``input_chunks = (flags, epoch, chunk)``: the inputs are still arriving by
    chunks of ``chunk`` systems; system i is read once ``flags[i // chunk] >=
    epoch`` (a CUDA int32 tensor raised behind each chunk's copy by SM-free
    work: copy engines / stream memory operations).  ``chunk_done`` (CUDA int32
    tensor) gets +1 per finished system of each chunk after its outputs are
    written (a copy stream can wait on it and read the chunk back early)."""
    a, b = as_device(a), as_device(b)
    precond, residual = as_device(precond), as_device(residual)
    batch, n, n2 = a.shape
    if n != n2 or n > 32:
        raise ValueError("batched path expects batch x n x n with n <= 32")
    if b.shape != (batch, n):
        raise ValueError("dimension mismatch")
    rates = tuple(int(x) for x in rates)
    if not rates or any(x < 1 for x in rates):
        raise ValueError("rates must be positive integers")
    if order_n < 1:
        raise ValueError("order_n must be >= 1")
    p_in = as_device(p).contiguous()
    f_in = as_device(f).contiguous()
    th_in = as_device(theta).contiguous()
    if p_in.shape != a.shape or f_in.shape != a.shape or th_in.shape != b.shape:
        raise ValueError("dimension mismatch")
    p_io, f_io, th_io = torch.empty_like(p_in), torch.empty_like(f_in), torch.empty_like(th_in)
    plans = [geometric_base_plan(x) if x > 1 else None for x in rates]
    code, offsets, consts = encode_many(plans)
    buf = _lib.counter_buf()
    flags_ptr, epoch, chunk = None, 0, 1
    if input_chunks is not None:
        flags, epoch, chunk = input_chunks
        if flags.dtype != torch.int32 or not flags.is_cuda or chunk < 1 or \
                flags.numel() < (batch + chunk - 1) // chunk:
            raise ValueError("input_chunks: a CUDA int32 flag per chunk and chunk >= 1")
        flags_ptr = flags.data_ptr()
    if chunk_done is not None and (chunk_done.dtype != torch.int32 or not chunk_done.is_cuda):
        raise ValueError("chunk_done must be a CUDA int32 tensor")
    if chunk_done is not None and input_chunks is None:
        raise ValueError("chunk_done needs input_chunks (only the gated kernel raises it)")
    if input_chunks is not None and iters < 1:
        raise ValueError("a gated call (input_chunks) needs iters >= 1")
    _lib.call("si_batched_composite_richardson_gated", _lib.handle(a.device.index), batch, n,
              a.data_ptr(), b.data_ptr(), precond.data_ptr(), residual.data_ptr(), len(rates),
              _lib.i32_array(list(rates)), _lib.i32_array(code), _lib.i64_array(offsets),
              _lib.f64_array(consts), len(consts), order_n, iters, p_in.data_ptr(),
              f_in.data_ptr(), th_in.data_ptr(), p_io.data_ptr(), f_io.data_ptr(),
              th_io.data_ptr(), flags_ptr, epoch, chunk,
              chunk_done.data_ptr() if chunk_done is not None else None, buf,
              _lib.stream_ptr(a.device))
    if ctr is not None:
        ctr.absorb(buf)
    return p_io, f_io, th_io


def batched_ns_richardson(a, b, p, f, theta, order: int, iters: int, plan=None,
                          ctr: MulCounter | None = None, out=None):
    """``iters`` x { plain Richardson with P_k; ns_step(order, plan) } for a batch of
    n x n systems (n <= 64) in one launch; BASELINE config 1 is batch = 1, n = 64,
    order 3.  Returns new (P, F, theta); inputs untouched.  ``out`` (optional):
    caller-owned contiguous device tensors (P', F', theta') of the input shapes
    to write into, e.g. views of one packed buffer for a single read-back."""
    from .series_toolkit import encode_plan

    a, b = as_device(a), as_device(b)
    squeeze = a.ndim == 2
    if squeeze:
        a, b = a[None], b.reshape(1, -1)
    batch, n, n2 = a.shape
    if n != n2 or n > 64:
        raise ValueError("batched path expects batch x n x n with n <= 64")
    if b.shape != (batch, n):
        raise ValueError("dimension mismatch")
    if order < 1:
        raise ValueError("order must be >= 1")
    if plan is not None and plan.order_h != order:
        raise ValueError(f"plan order {plan.order_h} != iteration order {order}")
    p_in = as_device(p).reshape(batch, n, n).contiguous()
    f_in = as_device(f).reshape(batch, n, n).contiguous()
    th_in = as_device(theta).reshape(batch, n).contiguous()
    if out is None:
        p_io, f_io, th_io = torch.empty_like(p_in), torch.empty_like(f_in), torch.empty_like(th_in)
    else:
        p_io, f_io, th_io = out
        for o, ref in ((p_io, p_in), (f_io, f_in), (th_io, th_in)):
            if (not isinstance(o, torch.Tensor) or o.numel() != ref.numel() or
                    o.dtype != torch.float64 or o.device != ref.device or not o.is_contiguous()):
                raise ValueError("out tensors must be contiguous float64 device tensors "
                                 "of the input shapes")
        p_io, f_io, th_io = (p_io.view(p_in.shape), f_io.view(f_in.shape),
                             th_io.view(th_in.shape))
    code, consts = encode_plan(plan) if plan is not None else ([], [])
    buf = _lib.counter_buf()
    _lib.call("si_batched_ns_richardson_ex", _lib.handle(a.device.index), batch, n, a.data_ptr(),
              b.contiguous().data_ptr(), order, _lib.i32_array(code) if code else None, len(code),
              _lib.f64_array(consts) if consts else None, len(consts), iters, p_in.data_ptr(),
              f_in.data_ptr(), th_in.data_ptr(), p_io.data_ptr(), f_io.data_ptr(),
              th_io.data_ptr(), buf, _lib.stream_ptr(a.device))
    if ctr is not None:
        ctr.absorb(buf)
    if squeeze:
        return p_io[0], f_io[0], th_io[0]
    return p_io, f_io, th_io
