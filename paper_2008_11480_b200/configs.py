"""Seeded synthetic inputs for the five BASELINE.json configs.

Host builders use numpy PCG64 (``default_rng(seed)``) with the draw order of
Appendix A, so the oracle and the device consume identical bits.  The device
builders (``*_device``) draw the same random numbers on the host but do the
O(n^3) assembly with the library's GEMM, for sizes where a host GEMM would
dominate setup (n >= 8192); their A differs from the host build only by GEMM
rounding, and parity at those sizes compares against an oracle fed the same
device-built A.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "c1_dense_small",
    "c2_batched",
    "c3_gram",
    "c4_householder",
    "c4_householder_device",
    "c5_gram_device",
]


def _sym(a):
    return (a + a.T) / 2.0


def c1_dense_small(n: int = 64, seed: int = 0):
    """A = Q diag(lambda) Q^T, Q = qr(N(0,1)), lambda log-uniform in [1, 100]; b ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    g0 = rng.standard_normal((n, n))
    q, _ = np.linalg.qr(g0)
    lam = np.exp(rng.uniform(0.0, np.log(100.0), n))
    b = rng.standard_normal(n)
    a = _sym((q * lam) @ q.T)
    return a, b


def c2_batched(batch: int = 16384, n: int = 32, m: int = 64, seed: int = 0):
    """A_i = G_i^T G_i / 64 + 1e-3 I with G_i a 64 x 32 Gaussian; one Gaussian RHS each.
    Draw order per system: G_i then b_i (one (m*n + n)-row block per system)."""
    rng = np.random.default_rng(seed)
    draws = rng.standard_normal((batch, m * n + n))
    g = draws[:, : m * n].reshape(batch, m, n)
    b = np.ascontiguousarray(draws[:, m * n :])
    a = np.einsum("bki,bkj->bij", g, g) / m + 1e-3 * np.eye(n)
    a = (a + np.transpose(a, (0, 2, 1))) / 2.0
    return np.ascontiguousarray(a), b


def c3_gram(n: int = 4096, m: int | None = None, seed: int = 0, shift: float = 1e-4):
    """A = G^T G / m + shift I with G an m x n Gaussian (m = 2n); b ~ N(0,1)."""
    m = 2 * n if m is None else m
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((m, n))
    b = rng.standard_normal(n)
    a = _sym(g.T @ g / m + shift * np.eye(n))
    return a, b


def _c4_draws(n: int, reflectors: int, rhs: int, seed: int):
    rng = np.random.default_rng(seed)
    lam = np.exp(rng.uniform(0.0, np.log(1e6), n))
    v = rng.standard_normal((reflectors, n))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    b = rng.standard_normal((n, rhs))
    return lam, v, b


def c4_householder(n: int = 16384, reflectors: int = 64, rhs: int = 64, seed: int = 0):
    """A = Q diag(lambda) Q^T, Q = H_1 ... H_64 (H_i = I - 2 v_i v_i^T),
    lambda log-uniform in [1, 1e6]; ``rhs`` Gaussian right-hand sides."""
    lam, v, b = _c4_draws(n, reflectors, rhs, seed)
    q = np.eye(n)
    for vi in v:
        q -= 2.0 * np.outer(q @ vi, vi)
    a = _sym((q * lam) @ q.T)
    return a, b


def c4_householder_device(n: int = 16384, reflectors: int = 64, rhs: int = 64, seed: int = 0):
    """Device build of :func:`c4_householder` (same draws; Q Lambda Q^T on the DMMA GEMM)."""
    import torch

    from . import _lib

    lam, v, b = _c4_draws(n, reflectors, rhs, seed)
    dev = torch.device("cuda", torch.cuda.current_device())
    q = torch.eye(n, dtype=torch.float64, device=dev)
    vt = torch.as_tensor(v, device=dev)
    for i in range(reflectors):
        vi = vt[i]
        q -= 2.0 * torch.outer(q @ vi, vi)
    ql = q * torch.as_tensor(lam, device=dev)[None, :]
    qt = q.T.contiguous()
    del q
    a = torch.empty((n, n), dtype=torch.float64, device=dev)
    _lib.call("si_gemm", _lib.handle(dev.index), n, n, n, 1.0, ql.data_ptr(), n, qt.data_ptr(), n,
              0.0, None, n, 0.0, a.data_ptr(), n, 0, None, _lib.stream_ptr(dev))
    del ql, qt
    out = torch.empty_like(a)
    _lib.call("si_symmetrize", _lib.handle(dev.index), n, a.data_ptr(), out.data_ptr(),
              _lib.stream_ptr(dev))
    return out, torch.as_tensor(b, device=dev)


def c5_gram_device(n: int = 32768, m: int = 40000, rhs: int = 256, seed: int = 0,
                   shift: float = 1e-3, chunk: int = 4096):
    """A = G^T G / m + shift I, G an m x n Gaussian drawn in row chunks on the host
    (PCG64, same order as one (m, n) draw), accumulated with the DMMA GEMM."""
    import torch

    from . import _lib

    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", torch.cuda.current_device())
    a = torch.zeros((n, n), dtype=torch.float64, device=dev)
    h, s = _lib.handle(dev.index), _lib.stream_ptr(dev)
    done = 0
    while done < m:
        rows = min(chunk, m - done)
        gc = torch.as_tensor(rng.standard_normal((rows, n)), device=dev)
        gt = gc.T.contiguous()
        _lib.call("si_gemm", h, n, n, rows, 1.0, gt.data_ptr(), rows, gc.data_ptr(), n, 1.0,
                  a.data_ptr(), n, 0.0, a.data_ptr(), n, 0, None, s)
        done += rows
    b = torch.as_tensor(rng.standard_normal((n, rhs)), device=dev)
    a /= m
    a += shift * torch.eye(n, dtype=torch.float64, device=dev)
    out = torch.empty_like(a)
    _lib.call("si_symmetrize", h, n, a.data_ptr(), out.data_ptr(), s)
    return out, b
