"""Degenerate and ragged inputs through the C ABI: empty products, K = 0, order-1
series, rate-1 parts, odd sizes that are not multiples of any tile."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _gemm(m, n, k, alpha=1.0, beta=0.0, diag=0.0, seed=0):
    from paper_2008_11480_b200 import _lib

    rng = np.random.default_rng(seed)
    a = torch.as_tensor(rng.standard_normal((m, max(k, 1)))[:, :k].copy(), device="cuda")
    b = torch.as_tensor(rng.standard_normal((max(k, 1), n))[:k].copy(), device="cuda")
    c = torch.as_tensor(rng.standard_normal((m, n)), device="cuda")
    d = torch.full((m, n), np.nan, dtype=torch.float64, device="cuda")
    buf = _lib.counter_buf()
    _lib.call("si_gemm", _lib.handle(), m, n, k, alpha, a.data_ptr() if a.numel() else c.data_ptr(),
              max(k, 1), b.data_ptr() if b.numel() else c.data_ptr(), max(n, 1), beta,
              c.data_ptr() if beta else None, max(n, 1), diag, d.data_ptr(), max(n, 1), 0, buf,
              _lib.stream_ptr())
    ref = alpha * (a.cpu().numpy() @ b.cpu().numpy()) + beta * c.cpu().numpy() + diag * np.eye(m, n)
    return d.cpu().numpy(), ref, buf


@pytest.mark.parametrize("m,n,k", [(0, 5, 3), (5, 0, 3), (130, 140, 0), (3, 3, 0)])
def test_empty_and_zero_depth_products(m, n, k):
    out, ref, buf = _gemm(m, n, k, beta=1.0, diag=1.0)
    assert out.shape == ref.shape
    assert np.array_equal(out, ref)  # K = 0: only the epilogue terms, exactly
    assert buf[0] == 1


@pytest.mark.parametrize("n", [1, 2, 3, 7, 33, 127, 129, 255, 257])
def test_ragged_sizes_through_a_step(n):
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as O

    rng = np.random.default_rng(n)
    g = rng.standard_normal((2 * n, n))
    a = g.T @ g / (2 * n) + 0.5 * np.eye(n)
    a = (a + a.T) / 2.0
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0)
    st = P.composite_step(P.initial_series(sp, 0, 1, order=2), sp.matrix, sp,
                          P.CompositeSpec((1, 2, 3)), 2)
    osp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    ost = O.composite_step(O.initial_series(osp, 0, 1, 2), osp.matrix, osp, (1, 2, 3), 2)
    err = np.linalg.norm(st.estimate.cpu().numpy() - ost.estimate) / np.linalg.norm(ost.estimate)
    assert err <= 1e-12
    assert st.ctr.mmm == ost.ctr.mmm


def test_order_one_degenerate_forms():
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as O

    rng = np.random.default_rng(2)
    g = rng.standard_normal((12, 6))
    a = g.T @ g / 12 + 0.5 * np.eye(6)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0)
    osp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    ctr = P.MulCounter()
    # Horner of order 1 is X itself, no product (series_toolkit.py:279-302)
    out = P.horner_eval(sp.residual, sp.precond, 1, ctr)
    assert torch.equal(out, sp.precond) and ctr.mmm == 0
    # geometric order 1 copies X (series_toolkit.py:448-449)
    out = P.geometric_apply(sp.residual, sp.precond, 1, sp.matrix, ctr)
    assert torch.equal(out, sp.precond) and ctr.mmm == 0
    # ns_step with order 1: G' = G, F' = I - G A (one product)
    st = P.initial_series(sp, 0, 1, order=1)
    st1 = P.ns_step(st, sp.matrix)
    ost1 = O.ns_step(O.initial_series(osp, 0, 1, 1), osp.matrix)
    assert np.allclose(st1.residual.cpu().numpy(), ost1.residual, atol=1e-15)
    assert st1.ctr.mmm == 1
    # composite with rate 1 and order_n = 1: G <- B G + S^-1 (newton_schulz test)
    stc = P.composite_step(st, sp.matrix, sp, P.CompositeSpec((1,)), 1)
    expected = sp.residual.cpu().numpy() @ sp.precond.cpu().numpy() + sp.precond.cpu().numpy()
    assert np.linalg.norm(stc.estimate.cpu().numpy() - expected) <= 1e-12 * np.linalg.norm(expected)


def test_exact_inverse_is_reproduced():
    """B = 0 (A diagonal): the composite part alone gives A^-1 exactly
    (reference test_newton_schulz.py:140-148)."""
    import paper_2008_11480_b200 as P

    a = np.diag([2.0, 4.0])
    sp = P.split_diagonal(a)
    st = P.composite_step(P.initial_series(sp, 0, 1, order=2), sp.matrix, sp,
                          P.CompositeSpec((3,)), 2)
    assert np.allclose(st.estimate.cpu().numpy(), np.diag([0.5, 0.25]), atol=1e-15)
    assert P.fro_norm(st.residual) <= 1e-15


def test_c_host_demo():
    """A non-Python host of the C ABI (examples/c_host_demo.c: split, initial
    series, plain Richardson + NS steps, norms, error status, the INT8-emulated
    backend, the sharded entry point) built by build()."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples",
                       "c_host_demo")
    assert os.path.exists(exe), "examples/c_host_demo not built (run build())"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bad-call status=-1" in out.stdout
    assert "sharded ns_step (NCCL, 1 rank) bitwise equal: yes" in out.stdout
    assert "ns_step emulated on the INT8 tensor cores vs FP64 DMMA: rel diff" in out.stdout


def test_batched_ns_richardson_into_packed_outputs():
    """``out=`` views of one packed buffer (the single read-back of bench.py's C1
    e2e path) hold exactly what the default outputs hold; bad ``out`` raises."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a_np, b_np = configs.c1_dense_small()
    a, b = P.as_device(a_np), P.as_device(b_np)
    alpha = float(torch.max(torch.sum(torch.abs(a), dim=1)))
    eye = torch.eye(64, dtype=torch.float64, device="cuda")
    p0, f0, t0 = eye / alpha, eye - a / alpha, torch.zeros_like(b)
    ref = P.batched_ns_richardson(a, b, p0, f0, t0, 3, 7)
    packed = torch.full((2 * 64 * 64 + 64,), float("nan"), dtype=torch.float64, device="cuda")
    got = P.batched_ns_richardson(a, b, p0, f0, t0, 3, 7,
                                  out=(packed[:4096], packed[4096:8192], packed[8192:]))
    torch.cuda.synchronize()
    for x, y in zip(got, ref):
        assert torch.equal(x, y)
    assert torch.equal(packed[:4096].view(64, 64), ref[0])
    assert torch.equal(packed[8192:], ref[2])
    with pytest.raises(ValueError):
        P.batched_ns_richardson(a, b, p0, f0, t0, 3, 7, out=(packed[:100], packed, packed))
