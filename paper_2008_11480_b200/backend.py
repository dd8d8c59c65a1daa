"""FP64 product backend of the device path (C ABI ``si_set_gemm_backend``).

Every n x n product of the hot path (``mat_mul``, matrix_core.py:101-106, and
the fused products of the series evaluators and steps) runs on one of two
tensor-core paths of the library:

* ``"dmma"`` (default): FP64 DMMA, TMA-fed (csrc/gemm_tma.cu).
* ``"ozaki"``: Ozaki scheme II (csrc/ozaki.cu) -- the product computed exactly
  from power-of-two-scaled integer images of A and B with one INT8 tcgen05 GEMM
  per modulus and recombined by the Chinese remainder theorem.  Used for
  products whose three dimensions are all >= ``min_dim``; the rest stay on
  DMMA.  Results are not bitwise the DMMA results: the error of an entry is
  bounded by ~2^-pa times the largest entries of its row of A and column of B
  (pa ~ 54 with 16 moduli at K = 16384), the same order as DGEMM's own.

The setting belongs to the device's library handle (all calls on that device).
"""

from __future__ import annotations

import contextlib
import ctypes

import torch

from . import _lib

_NAMES = {"dmma": 0, "ozaki": 1}


def set_gemm_backend(name: str, moduli: int = 0, min_dim: int = 0,
                     device: int | None = None) -> None:
    """Select the FP64 product backend; ``moduli`` (8..16) and ``min_dim``
    (>= 128) keep their current values when 0."""
    if name not in _NAMES:
        raise ValueError(f"unknown GEMM backend {name!r} (expected one of {sorted(_NAMES)})")
    _lib.call("si_set_gemm_backend", _lib.handle(device), _NAMES[name], int(moduli), int(min_dim))


def get_gemm_backend(device: int | None = None) -> tuple[str, int, int]:
    """(name, moduli, min_dim) of the device's handle."""
    b, m, d = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    _lib.call("si_get_gemm_backend", _lib.handle(device), ctypes.byref(b), ctypes.byref(m),
              ctypes.byref(d))
    name = {v: k for k, v in _NAMES.items()}[b.value]
    return name, m.value, d.value


@contextlib.contextmanager
def gemm_backend(name: str, moduli: int = 0, min_dim: int = 0, device: int | None = None):
    """Temporarily select a backend (restored on exit)."""
    prev = get_gemm_backend(device)
    set_gemm_backend(name, moduli, min_dim, device)
    try:
        yield
    finally:
        set_gemm_backend(prev[0], prev[1], prev[2], device)


def set_ozaki_chunks(max_rows: int = 0, max_cols: int = 0, device: int | None = None) -> None:
    """Bound the emulated products' workspace: D in chunks of at most
    ``max_rows`` x ``max_cols`` (multiples of 256; 0 = automatic).  Results do
    not depend on the chunking (bitwise)."""
    if max_rows < 0 or max_cols < 0:
        raise ValueError("chunk bounds must be >= 0")
    _lib.call("si_set_ozaki_chunks", _lib.handle(device), int(max_rows), int(max_cols))


_KERNELS = {"auto": 0, "pair": 1, "single": 2, "multicast": 3}


def set_ozaki_kernel(name: str, device: int | None = None) -> None:
    """INT8 tensor-core kernel of the emulated products: ``"single"`` (one CTA
    per 128 x 256 tile; what ``"auto"`` picks) or ``"pair"`` (2-CTA clusters,
    tcgen05.mma.cta_group::2, 256 x 256 tiles).  Results are identical."""
    if name not in _KERNELS:
        raise ValueError(f"unknown INT8 kernel {name!r} (expected one of {sorted(_KERNELS)})")
    _lib.call("si_set_ozaki_kernel", _lib.handle(device), _KERNELS[name])


def ozaki_moduli(n: int = 16) -> list[int]:
    """The first ``n`` moduli of the emulation (pairwise coprime, <= 256)."""
    out = (ctypes.c_uint32 * n)()
    _lib.call("si_ozaki_moduli", int(n), out)
    return list(out)


def i8_gemm_mod(a: torch.Tensor, bt: torch.Tensor) -> torch.Tensor:
    """The INT8 tensor-core kernel alone: ``r[l] = (a[l] @ bt[l].T) mod m_l``.

    ``a``: (planes, m, kp) int8, ``bt``: (planes, n, kp) int8 (kp a multiple of
    128), both contiguous CUDA tensors; returns (planes, m, n) uint8."""
    if a.dtype != torch.int8 or bt.dtype != torch.int8 or a.dim() != 3 or bt.dim() != 3:
        raise ValueError("a and bt must be 3-d int8 tensors")
    if a.shape[0] != bt.shape[0] or a.shape[2] != bt.shape[2]:
        raise ValueError("a and bt must agree in planes and kp")
    a = a.contiguous()
    bt = bt.contiguous()
    p, m, kp = a.shape
    n = bt.shape[1]
    r = torch.empty((p, m, n), dtype=torch.uint8, device=a.device)
    _lib.call("si_i8_gemm_mod", _lib.handle(a.device.index), _lib.ptr(a), _lib.ptr(bt), _lib.ptr(r),
              m, n, kp, p, _lib.stream_ptr(a.device))
    return r
