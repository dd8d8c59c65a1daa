"""Device-resident counterpart of ``seriesinv.matrix_core`` (matrix_core.py).

Matrices are contiguous float64 CUDA tensors.  ``mat_mul`` / ``mat_vec`` run the
library's DMMA kernels through ``si_gemm`` and tick the same :class:`MulCounter`
fields as the reference (matrix_core.py:71-114), so cost comparisons carry
over unchanged.  Nothing here computes on the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _lib

__all__ = [
    "MulCounter",
    "Norms",
    "SpectralRadiusError",
    "as_device",
    "fro_norm",
    "identity",
    "inf_norm",
    "load_matrix",
    "load_vector",
    "mat_mul",
    "mat_pow",
    "mat_pow_counted",
    "mat_vec",
    "norms",
    "save_matrix",
    "save_vector",
    "spectral_radius",
    "square_matrix",
    "to_host",
    "vector",
]


@dataclass
class MulCounter:
    """Tally of matrix-matrix (mmm) and matrix-vector (mvm) products
    (matrix_core.py:71-98).  Branches merged by summation."""

    mmm: int = 0
    mvm: int = 0

    def count_mmm(self, n: int = 1) -> None:
        if n < 0:
            raise ValueError("counter increments must be non-negative")
        self.mmm += n

    def count_mvm(self, n: int = 1) -> None:
        if n < 0:
            raise ValueError("counter increments must be non-negative")
        self.mvm += n

    def merge(self, other: "MulCounter") -> None:
        self.mmm += other.mmm
        self.mvm += other.mvm

    def copy(self) -> "MulCounter":
        return MulCounter(self.mmm, self.mvm)

    def absorb(self, buf) -> None:
        """Add a native ``int64[2]`` counter delta."""
        self.mmm += int(buf[0])
        self.mvm += int(buf[1])


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.NativeUnavailable("no CUDA device visible: the seriesinv B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def as_device(x, device: torch.device | None = None) -> torch.Tensor:
    """float64, contiguous, on the current CUDA device (copies only if needed)."""
    # fast path (small-system calls are host-bound): already a contiguous
    # float64 tensor on the current device -- returned as is, no dispatch
    if (isinstance(x, torch.Tensor) and x.dtype == torch.float64 and x.is_cuda
            and x.is_contiguous()
            and x.device.index == (torch.cuda.current_device() if device is None
                                   else device.index)):
        return x
    dev = device or _device()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=dev)


def to_host(x: torch.Tensor) -> np.ndarray:
    return x.detach().to("cpu").numpy()


def square_matrix(entries) -> torch.Tensor:
    """Validate a square, finite matrix (matrix_core.py:40-53) and place it on the device."""
    t = as_device(entries)
    if t.ndim != 2 or t.shape[0] != t.shape[1] or t.shape[0] < 1:
        raise ValueError(f"expected a square matrix, got shape {tuple(t.shape)}")
    if not bool(torch.isfinite(t).all()):
        raise ValueError("matrix entries must be finite")
    return t


def vector(entries) -> torch.Tensor:
    """Validate a finite vector (matrix_core.py:56-64)."""
    t = as_device(entries).reshape(-1)
    if t.numel() < 1:
        raise ValueError("vector must have at least one entry")
    if not bool(torch.isfinite(t).all()):
        raise ValueError("vector entries must be finite")
    return t


def identity(dim: int) -> torch.Tensor:
    return torch.eye(dim, dtype=torch.float64, device=_device())


def _gemm(a: torch.Tensor, b: torch.Tensor, is_mv: bool, ctr: MulCounter | None) -> torch.Tensor:
    a = as_device(a)
    b = as_device(b)
    vec = b.ndim == 1
    b2 = b.reshape(-1, 1) if vec else b
    if a.shape[1] != b2.shape[0]:
        raise ValueError(f"dimension mismatch: {tuple(a.shape)} @ {tuple(b.shape)}")
    m, k = a.shape
    n = b2.shape[1]
    out = torch.empty((m, n), dtype=torch.float64, device=a.device)
    buf = _lib.counter_buf()
    _lib.call(
        "si_gemm", _lib.handle(a.device.index), m, n, k, 1.0, a.data_ptr(), k, b2.data_ptr(), n,
        0.0, None, n, 0.0, out.data_ptr(), n, int(is_mv), buf, _lib.stream_ptr(a.device),
    )
    if ctr is not None:
        ctr.absorb(buf)
    return out.reshape(-1) if vec else out


def mat_mul(a, b, ctr: MulCounter) -> torch.Tensor:
    """``a @ b`` on the DMMA kernels; ``ctr.mmm += 1`` (matrix_core.py:101-106)."""
    return _gemm(a, b, False, ctr)


def mat_vec(a, v, ctr: MulCounter) -> torch.Tensor:
    """``a @ v`` (v may be n x r); ``ctr.mvm += 1`` (matrix_core.py:109-114)."""
    return _gemm(a, v, True, ctr)


def mat_pow_counted(a, e: int, ctr: MulCounter) -> torch.Tensor:
    """Binary exponentiation, every product counted (matrix_core.py:137-151)."""
    if e < 0:
        raise ValueError("exponent must be non-negative")
    a = as_device(a)
    out = torch.empty_like(a)
    buf = _lib.counter_buf()
    _lib.call("si_mat_pow_counted", _lib.handle(a.device.index), a.shape[0], a.data_ptr(), int(e),
              out.data_ptr(), buf, _lib.stream_ptr(a.device))
    ctr.absorb(buf)
    return out


def mat_pow(a, e: int) -> torch.Tensor:
    """Uncounted ``a**e`` (matrix_core.py:117-134)."""
    return mat_pow_counted(a, e, MulCounter())


class Norms(NamedTuple):
    frobenius: float
    inf_norm: float


def fro_norm(a) -> float:
    a = as_device(a)
    a2 = a.reshape(a.shape[0], -1) if a.ndim != 1 else a.reshape(-1, 1)
    out = ctypes.c_double()
    _lib.call("si_fro_norm", _lib.handle(a.device.index), a2.shape[0], a2.shape[1], a2.data_ptr(),
              a2.shape[1], ctypes.byref(out), _lib.stream_ptr(a.device))
    return float(out.value)


def inf_norm(a) -> float:
    a = as_device(a)
    a2 = a.reshape(a.shape[0], -1) if a.ndim != 1 else a.reshape(-1, 1)
    out = ctypes.c_double()
    _lib.call("si_inf_norm", _lib.handle(a.device.index), a2.shape[0], a2.shape[1], a2.data_ptr(),
              a2.shape[1], ctypes.byref(out), _lib.stream_ptr(a.device))
    return float(out.value)


def norms(a) -> Norms:
    """Frobenius and infinity norms (matrix_core.py:154-172)."""
    return Norms(frobenius=fro_norm(a), inf_norm=inf_norm(a))


# ---------------------------------------------------------------------------
# On-disk formats: the reference's text format (matrix_core.py:242-310: a "dim"
# line, then rows, '#' comment lines, 17 significant digits) and a binary .npy
# path for the sizes where text is unusable (25 GB of text at n=32768).
# ---------------------------------------------------------------------------


def _data_lines(text: str) -> list[str]:
    return [ln.strip() for ln in text.splitlines() if ln.strip() and not ln.strip().startswith("#")]


def load_matrix(path, device: torch.device | None = None) -> torch.Tensor:
    """Square matrix from ``.npy`` or the reference text format, placed on the device."""
    if str(path).endswith(".npy"):
        return square_matrix(np.load(path, allow_pickle=False))
    with open(path, "r", encoding="utf-8") as fh:
        lines = _data_lines(fh.read())
    if not lines:
        raise ValueError(f"{path}: empty matrix file")
    dim = int(lines[0])
    if dim < 1:
        raise ValueError(f"{path}: dimension must be positive, got {dim}")
    if len(lines) != 1 + dim:
        raise ValueError(f"{path}: expected {dim} data rows, got {len(lines) - 1}")
    rows = []
    for i, line in enumerate(lines[1:]):
        row = [float(tok) for tok in line.split()]
        if len(row) != dim:
            raise ValueError(f"{path}: row {i} has {len(row)} entries, expected {dim}")
        rows.append(row)
    return square_matrix(np.array(rows))


def save_matrix(path, a, comment: str | None = None) -> None:
    """Write ``.npy`` (binary) or the reference text format (17 significant digits)."""
    host = to_host(a) if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    if host.ndim != 2 or host.shape[0] != host.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {host.shape}")
    if str(path).endswith(".npy"):
        np.save(path, host)
        return
    with open(path, "w", encoding="utf-8") as fh:
        for line in (comment or "").splitlines():
            fh.write(f"# {line}\n")
        fh.write(f"{host.shape[0]}\n")
        for row in host:
            fh.write(" ".join(format(x, ".17g") for x in row) + "\n")


def load_vector(path) -> torch.Tensor:
    if str(path).endswith(".npy"):
        return vector(np.load(path, allow_pickle=False))
    with open(path, "r", encoding="utf-8") as fh:
        lines = _data_lines(fh.read())
    if not lines:
        raise ValueError(f"{path}: empty vector file")
    dim = int(lines[0])
    values = [float(tok) for line in lines[1:] for tok in line.split()]
    if len(values) != dim:
        raise ValueError(f"{path}: expected {dim} entries, got {len(values)}")
    return vector(values)


def save_vector(path, v, comment: str | None = None) -> None:
    host = to_host(v) if isinstance(v, torch.Tensor) else np.asarray(v, dtype=np.float64)
    host = host.reshape(-1)
    if str(path).endswith(".npy"):
        np.save(path, host)
        return
    with open(path, "w", encoding="utf-8") as fh:
        for line in (comment or "").splitlines():
            fh.write(f"# {line}\n")
        fh.write(f"{host.size}\n")
        for x in host:
            fh.write(format(x, ".17g") + "\n")


class SpectralRadiusError(RuntimeError):
    """Power iteration failed to settle; carries the best estimate seen (matrix_core.py:175-180)."""

    def __init__(self, message: str, best_estimate: float):
        super().__init__(message)
        self.best_estimate = best_estimate


def spectral_radius(a, tol: float = 1e-12, max_iter: int = 10000, seed: int = 0,
                    check_every: int = 32) -> float:
    """Norm-ratio power iteration (matrix_core.py:183-239).

    The iteration runs on the device (``si_power_iterate``: GEMV, norm, the
    reference's streak rule and x = y / est in kernels, no host round trip per
    iteration); the host looks at the state every ``check_every`` iterations.
    Start and restart vectors are the reference's draws (``default_rng(seed)``
    normals, normalised on the host), so the sequence of estimates is the
    reference's up to GEMV rounding."""
    a = as_device(a)
    dim = a.shape[0]
    if a.ndim != 2 or a.shape != (dim, dim):
        raise ValueError("spectral_radius expects a square matrix")
    a = a.contiguous()
    rng = np.random.default_rng(seed)

    def fresh():
        x = rng.standard_normal(dim)
        return as_device(x / np.linalg.norm(x))

    best, restarts, used = 0.0, 0, 0
    x = fresh()
    h, s = _lib.handle(a.device.index), _lib.stream_ptr(a.device)
    while used < max_iter:
        est, bst = ctypes.c_double(), ctypes.c_double()
        its, status = ctypes.c_int64(), ctypes.c_int()
        _lib.call("si_power_iterate", h, dim, a.data_ptr(), dim, x.data_ptr(), float(tol),
                  max_iter - used, int(check_every), ctypes.byref(est), ctypes.byref(bst),
                  ctypes.byref(its), ctypes.byref(status), s)
        used += its.value
        if bst.value != 0.0:
            best = bst.value
        if status.value == 1:
            return est.value
        if status.value == 2:
            # est == 0: x is (numerically) in the null space (matrix_core.py:203-215)
            if fro_norm(a) == 0.0:
                return 0.0
            restarts += 1
            if restarts > 3:
                return 0.0
            x = fresh()
            continue
        break
    raise SpectralRadiusError(
        f"power iteration did not converge within {max_iter} iterations (best estimate {best:.6e})",
        best_estimate=best,
    )
