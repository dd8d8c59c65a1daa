"""Newton-Schulz steps on the device: the behaviours the
reference's NS tests pin -- the exponent laws of the classical, composite,
double and additive steps (F_k = B^e), step costs, plan / spec / order
validation, exact inverses, rate presets, the doubling path for large rates,
executor bitwise equality and the stop rule."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _sdd(dim, rho, rng, jitter=0.002):
    """Symmetric SDD matrix whose diagonal splitting has rho(B) ~= rho."""
    w = rng.uniform(0.5, 1.5, (dim, dim))
    w = (w + w.T) / 2.0
    np.fill_diagonal(w, 0.0)
    for _ in range(200):
        s = np.sqrt(w.sum(axis=1) / rho)
        w = w / np.outer(s, s)
    return np.diag(1.0 + jitter * rng.uniform(0.0, 1.0, dim)) - w


def _system(dim, rho, seed):
    import paper_2008_11480_b200 as P

    a = P.square_matrix(_sdd(dim, rho, np.random.default_rng(seed)))
    return a, P.split_diagonal(a)


def _power_law(f, b, e, rel):
    target = np.linalg.matrix_power(_np(b), e)
    scale = np.linalg.norm(target)
    if scale < 1e-250:
        assert np.linalg.norm(_np(f)) <= 1e-200
    else:
        assert np.linalg.norm(_np(f) - target) <= rel * scale


def _consistent(st, a):
    n = a.shape[0]
    check = np.eye(n) - _np(st.estimate) @ _np(a)
    assert np.linalg.norm(check - _np(st.residual)) <= 1e-10 * (1 + np.linalg.norm(
        _np(st.residual)))


def test_initial_series():
    import paper_2008_11480_b200 as P

    a, sp = _system(4, 0.9, 0)
    st = P.initial_series(sp, 0, 1)
    assert torch.equal(st.estimate, sp.precond) and torch.equal(st.residual, sp.residual)
    assert (st.step, st.series_order, st.ctr.mmm) == (0, 1, 0)
    spi = P.split_diagonal(np.eye(3))
    for p, w in ((0, 1), (1, 2), (2, 2)):
        s = P.initial_series(spi, p, w)
        assert np.allclose(_np(s.estimate), np.eye(3), atol=1e-15)
        assert np.allclose(_np(s.residual), 0.0, atol=1e-15)
    a3, sp3 = _system(3, 0.9, 1)
    _power_law(P.initial_series(sp3, 1, 2).residual, sp3.residual, 4, 1e-12)
    _consistent(P.initial_series(sp, 2, 3), a)


def test_classical_step():
    import paper_2008_11480_b200 as P

    a, sp = _system(4, 0.95, 2)
    _power_law(P.ns_step(P.initial_series(sp, 0, 1, order=2), a).residual, sp.residual, 2,
               1e-12)
    st = P.initial_series(sp, 0, 1, order=2)
    for _ in range(3):
        st = P.ns_step(st, a)
    _power_law(st.residual, sp.residual, 8, 1e-9)
    st = P.initial_series(sp, 1, 1, order=3)            # h = 2
    for _ in range(2):
        st = P.ns_step(st, a)
    _power_law(st.residual, sp.residual, 18, 1e-9)
    for n in (2, 3, 5):                                  # cost = the order
        st = P.initial_series(sp, 0, 1, order=n)
        before = st.ctr.mmm
        assert P.ns_step(st, a).ctr.mmm - before == n
    plain = P.ns_step(P.initial_series(sp, 0, 1, order=8), a)
    plan = P.plan_order(8)
    st = P.initial_series(sp, 0, 1, order=8)
    before = st.ctr.mmm
    planned = P.ns_step(st, a, plan=plan)
    assert np.linalg.norm(_np(planned.estimate) - _np(plain.estimate)) <= 1e-10 * np.linalg.norm(
        _np(plain.estimate))
    assert planned.ctr.mmm - before == plan.mmm_poly + 1
    with pytest.raises(ValueError):
        P.ns_step(P.initial_series(sp, 0, 1, order=3), a, plan=P.plan_order(4))
    st = P.initial_series(sp, 1, 2, order=2)
    for _ in range(4):
        st = P.ns_step(st, a)
        _consistent(st, a)


def test_composite_step():
    import paper_2008_11480_b200 as P

    a, sp = _system(4, 0.9, 3)
    st = P.initial_series(sp, 0, 1, order=1)
    expected = _np(sp.precond)
    for _ in range(3):                                   # rates (1,), n = 1: G <- B G + S^-1
        st = P.composite_step(st, a, sp, P.CompositeSpec((1,)), order_n=1)
        expected = _np(sp.residual) @ expected + _np(sp.precond)
        assert np.linalg.norm(_np(st.estimate) - expected) <= 1e-11 * np.linalg.norm(expected)
    a, sp = _system(4, 0.95, 4)
    st = P.composite_step(P.initial_series(sp, 0, 1, order=2), a, sp, P.CompositeSpec((2, 3)), 2)
    _power_law(st.residual, sp.residual, 7, 1e-11)       # B^(5 + 2)
    d = P.square_matrix(np.diag([2.0, 4.0]))             # B = 0: exact inverse
    spd = P.split_diagonal(d)
    st = P.composite_step(P.initial_series(spd, 0, 1, order=2), d, spd, P.CompositeSpec((3,)), 2)
    assert np.allclose(_np(st.estimate), np.diag([0.5, 0.25]), atol=1e-15)
    assert P.fro_norm(st.residual) <= 1e-15
    a, sp = _system(4, 0.97, 5)
    st = P.initial_series(sp, 1, 1, order=2)             # h = 2
    e = 2
    for _ in range(2):
        st = P.composite_step(st, a, sp, P.CompositeSpec((2, 2)), 2)
        e = 4 + 2 * e
        _power_law(st.residual, sp.residual, e, 1e-9)
    assert e == P.composite_exponent(2, 2, 2, (2, 2))
    with pytest.raises(ValueError):
        P.CompositeSpec(())
    with pytest.raises(ValueError):
        P.CompositeSpec((0, 2))
    assert P.constant_rates(3, 2).rates == (3, 3)
    stepper = P.power_rates(2, 3)
    assert stepper(0).rates == (1, 1, 1) and stepper(3).rates == (8, 8, 8)
    with pytest.raises(ValueError):
        P.power_rates(1, 2)
    a, sp = _system(4, 0.995, 6)                         # rates m^k per step
    stepper = P.power_rates(2, 2)
    st = P.initial_series(sp, 0, 1, order=2)
    e = 1
    for k in range(1, 4):
        st = P.composite_step(st, a, sp, stepper(k), 2)
        e = 2 * 2 ** k + 2 * e
        _power_law(st.residual, sp.residual, e, 1e-9)
    a, sp = _system(4, 0.999, 7)                         # rate 100: the doubling path
    st = P.composite_step(P.initial_series(sp, 0, 1, order=2), a, sp, P.CompositeSpec((100,)), 2)
    _power_law(st.residual, sp.residual, 102, 1e-9)


def test_double_step():
    import paper_2008_11480_b200 as P

    a, sp = _system(4, 0.9, 8)
    st = P.initial_double(sp, 1, 2, order=2)
    n = 4
    assert np.linalg.norm((np.eye(n) - _np(st.accel_estimate) @ _np(a))
                          - _np(st.accel_residual)) <= 1e-10 * (1 + P.fro_norm(st.accel_residual))
    _consistent(st, a)
    a, sp = _system(4, 0.95, 9)
    _power_law(P.double_ns_step(P.initial_double(sp, 0, 1, order=2), a).residual, sp.residual, 6,
               1e-11)
    a, sp = _system(4, 0.97, 10)
    st = P.initial_double(sp, 0, 1, order=2)
    for _ in range(2):
        st = P.double_ns_step(st, a)
    _power_law(st.residual, sp.residual, 20, 1e-9)
    spi = P.split_diagonal(np.eye(3))
    st = P.initial_double(spi, 0, 1, order=2)
    assert np.allclose(_np(st.estimate), np.eye(3), atol=1e-15)
    assert P.fro_norm(P.double_ns_step(st, P.square_matrix(np.eye(3))).residual) <= 1e-15
    a, sp = _system(5, 0.95, 11)
    serial = P.initial_double(sp, 1, 2, order=3)
    threaded = P.initial_double(sp, 1, 2, order=3)
    with ThreadPoolExecutor(max_workers=2) as pool:
        for _ in range(3):
            serial = P.double_ns_step(serial, a)
            threaded = P.double_ns_step(threaded, a, executor=pool)
    for f in ("estimate", "residual", "accel_estimate"):
        assert torch.equal(getattr(serial, f), getattr(threaded, f))
    assert serial.ctr.mmm == threaded.ctr.mmm


def test_additive_step():
    import paper_2008_11480_b200 as P

    d = P.square_matrix(np.diag([2.0, 5.0]))
    exact = P.as_device(np.diag([0.5, 0.2]))
    z, g = P.additive_correction_step(exact, exact, d, 2, P.MulCounter())
    assert np.allclose(_np(g), np.diag([0.5, 0.2]), atol=1e-15)
    assert np.allclose(_np(z), np.diag([0.5, 0.2]), atol=1e-15)
    a, sp = _system(4, 0.95, 12)
    st = P.initial_series(sp, 0, 1)
    z, g = P.additive_correction_step(st.estimate, st.estimate, a, 2, st.ctr)
    _power_law(np.eye(4) - _np(z) @ _np(a), sp.residual, 2, 1e-11)
    _power_law(np.eye(4) - _np(g) @ _np(a), sp.residual, 3, 1e-11)
    a, sp = _system(4, 0.97, 13)
    st = P.initial_series(sp, 0, 1)
    z = g = st.estimate
    for _ in range(2):
        z, g = P.additive_correction_step(z, g, a, 3, st.ctr)
    _power_law(np.eye(4) - _np(z) @ _np(a), sp.residual, 9, 1e-10)
    _power_law(np.eye(4) - _np(g) @ _np(a), sp.residual, 13, 1e-10)
    assert P.additive_exponents(2, 3, 1) == (9, 13)
    with pytest.raises(ValueError):
        P.additive_correction_step(sp.precond, sp.precond, a, 1, P.MulCounter())


def test_stop_rule():
    import paper_2008_11480_b200 as P

    a, sp = _system(4, 0.5, 14)
    st = P.initial_series(sp, 0, 1, order=4)
    assert not P.converged(st)
    for _ in range(6):
        st = P.ns_step(st, a)
    assert P.converged(st)
    st = P.run_until_converged(P.initial_series(sp, 0, 1, order=3), a)
    assert P.converged(st) and st.step <= 30
    assert P.run_until_converged(P.initial_series(sp, 0, 1, order=2), a, max_steps=1).step == 1
