"""Fused stop-rule norm: ||F_k||_F^2 of a step's residual output from the
epilogues of the products that wrote F_k (si_set_step_norm; converged(),
newton_schulz.py:328-331 over fro_norm, matrix_core.py:167-168).

Checked against the separate reduction pass (si_fro_norm) on every producer
path: the FP64 DMMA GEMM epilogue, the CRT epilogue of the emulated products
(unchunked and row x column chunked), the small-n kernels (one partial pass),
the row-chunked residual of the e2e step, and a copied F (h = 1).  The slots
are reduced in a fixed order, so the value is bitwise reproducible.
"""

import pytest
import torch

import paper_2008_11480_b200 as P
from paper_2008_11480_b200 import _lib

pytestmark = pytest.mark.gpu

REL = 1e-13  # two summation orders of the same n^2 squares


def _spd(n, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(n, 2 * n, dtype=torch.float64, generator=g)
    return (x @ x.T / (2 * n) + 0.5 * torch.eye(n, dtype=torch.float64)).cuda()


def _check(st):
    assert st.residual_fro2 is not None
    fused = float(st.residual_fro2.item()) ** 0.5
    ref = P.fro_norm(st.residual)
    assert abs(fused - ref) <= REL * ref, (fused, ref)
    return fused


@pytest.mark.parametrize("n", [96, 300, 1024])
@pytest.mark.parametrize("backend", ["dmma", "ozaki"])
def test_ns_and_composite_steps(n, backend):
    with P.gemm_backend(backend, 16, 256):
        sp = P.split_scalar(_spd(n), check_pd=False, verify=False)
        st = P.initial_series(sp, 1, 1)
        _check(st)
        st1 = P.ns_step(st, sp.matrix)
        _check(st1)
        st2 = P.composite_step(st1, sp.matrix, sp, P.CompositeSpec((2, 3)), 2)
        f2 = _check(st2)
        again = P.composite_step(st1, sp.matrix, sp, P.CompositeSpec((2, 3)), 2)
        assert torch.equal(again.residual_fro2, st2.residual_fro2)  # fixed-order slots
        assert f2 < _check(st1)
        assert P.converged(st2) == (P.fro_norm(st2.residual) <= 1e-13 * n ** 0.5)


def test_emulated_chunked_products():
    n = 1536
    with P.gemm_backend("ozaki", 16, 256):
        sp = P.split_scalar(_spd(n, 1), check_pd=False, verify=False)
        st = P.ns_step(P.initial_series(sp, 1, 1), sp.matrix)
        P.set_ozaki_chunks(512, 768)
        try:
            st_c = P.ns_step(P.initial_series(sp, 1, 1), sp.matrix)
        finally:
            P.set_ozaki_chunks(0, 0)
        assert torch.equal(st_c.residual, st.residual)  # chunking is bitwise neutral
        _check(st_c)


def test_copied_residual_and_double_step():
    sp = P.split_scalar(_spd(200, 2), check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1)  # h = 1: F_0 is a copy of B, no product wrote it
    assert torch.equal(st.residual, sp.residual)
    _check(st)
    ds = P.initial_double(sp, 1, 1, 2)
    _check(ds)
    ds1 = P.double_ns_step(ds, sp.matrix)
    _check(ds1)
    ds1c = P.double_ns_step(ds, sp.matrix, executor=object())
    assert torch.equal(ds1c.residual_fro2, ds1.residual_fro2)


@pytest.mark.parametrize("backend", ["dmma", "ozaki"])
def test_row_chunked_residual(backend):
    n = 1024
    with P.gemm_backend(backend, 16, 256):
        sp = P.split_scalar(_spd(n, 3), check_pd=False, verify=False)
        st = P.initial_series(sp, 1, 1)
        ref = P.composite_step(st, sp.matrix, sp, P.CompositeSpec((2, 3)), 2)
        chunks = [torch.cuda.Event() for _ in range(4)]
        out = P.composite_step(st, sp.matrix, sp, P.CompositeSpec((2, 3)), 2,
                               residual_chunks=chunks)
        assert torch.equal(out.residual, ref.residual)
        _check(out)


def test_one_shot_target_is_consumed():
    h = _lib.handle(0)
    sp = P.split_scalar(_spd(128, 4), check_pd=False, verify=False)
    st = P.initial_series(sp, 1, 1)
    sentinel = torch.full((1,), -1.0, dtype=torch.float64, device="cuda")
    _lib.call("si_set_step_norm", h, sentinel.data_ptr())
    a = sp.matrix
    g, f = torch.empty_like(a), torch.empty_like(a)
    buf = _lib.counter_buf()
    s = _lib.stream_ptr(a.device)
    _lib.call("si_ns_step", h, 128, a.data_ptr(), st.estimate.data_ptr(), st.residual.data_ptr(),
              2, None, 0, None, 0, g.data_ptr(), f.data_ptr(), buf, s)
    torch.cuda.synchronize()
    assert abs(sentinel.item() ** 0.5 - P.fro_norm(f)) <= REL * P.fro_norm(f)
    sentinel.fill_(-1.0)
    _lib.call("si_ns_step", h, 128, a.data_ptr(), st.estimate.data_ptr(), st.residual.data_ptr(),
              2, None, 0, None, 0, g.data_ptr(), f.data_ptr(), buf, s)
    torch.cuda.synchronize()
    assert sentinel.item() == -1.0  # consumed by the first call
    # a failing step call from Python disarms the target
    with pytest.raises(ValueError):
        P.ns_step(st, sp.matrix[:64, :64])
    st1 = P.ns_step(st, sp.matrix)
    _check(st1)
