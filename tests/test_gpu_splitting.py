"""Splitting on the device (splitting.py:42-146): the behaviours
the reference's own splitting tests pin -- exact diagonal splits, spectral
radii, the eps and definiteness checks, the construction invariant
S^-1 A + B = I, the 2S - A criterion and the measured rho hint."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _spd(n, rng):
    m = rng.standard_normal((n, n))
    return m @ m.T / n + 0.5 * np.eye(n)


def _sdd(n, rng, margin=0.3):
    a = rng.uniform(-1.0, 1.0, (n, n))
    a = (a + a.T) / 2.0
    np.fill_diagonal(a, 0.0)
    np.fill_diagonal(a, np.abs(a).sum(axis=1) + margin)
    return a


def test_diagonal_split_cases():
    import paper_2008_11480_b200 as P

    sp = P.split_diagonal(P.square_matrix(np.diag([4.0, 9.0])))
    assert np.array_equal(_np(sp.residual), np.zeros((2, 2)))
    assert np.allclose(_np(sp.precond), np.diag([0.25, 1.0 / 9.0]), rtol=1e-15)
    sp = P.split_diagonal(P.square_matrix([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(_np(sp.residual), [[0.0, -0.5], [-0.5, 0.0]], atol=1e-15)
    assert P.spectral_radius(sp.residual) == pytest.approx(0.5, rel=1e-9)
    with pytest.raises(P.NotSDDError):
        P.split_diagonal(P.square_matrix([[1.0, 2.0], [2.0, 1.0]]))   # not dominant
    with pytest.raises(P.NotSDDError):
        P.split_diagonal(P.square_matrix([[-3.0, 1.0], [1.0, 3.0]]))  # negative diagonal
    with pytest.raises(ValueError):
        P.split_diagonal(P.square_matrix([[3.0, 1.0], [0.0, 3.0]]))   # not symmetric


def test_scalar_split_cases():
    import paper_2008_11480_b200 as P

    sp = P.split_scalar(np.eye(2), eps=1.0)            # alpha = 1/2 + 1
    assert np.allclose(_np(sp.precond), np.eye(2) / 1.5, rtol=1e-15)
    assert np.allclose(_np(sp.residual), np.eye(2) / 3.0, rtol=1e-14)
    assert np.allclose(_np(P.split_scalar(np.eye(2), eps=0.5).residual), 0.0, atol=1e-15)
    sp = P.split_scalar(P.square_matrix([[2.0, 1.0], [1.0, 2.0]]), eps=0.1)
    assert P.spectral_radius(sp.residual) == pytest.approx(0.875, rel=1e-9)  # |1 - 3/1.6|
    for eps in (0.0, -1.0):
        with pytest.raises(ValueError):
            P.split_scalar(np.eye(2), eps=eps)
    with pytest.raises(P.NotSPDError):
        P.split_scalar(P.square_matrix([[1.0, 2.0], [2.0, 1.0]]), eps=0.1)
    a = _spd(4, np.random.default_rng(0))
    sp = P.split_scalar(a)                               # default eps = 1e-3 ||A||_inf
    alpha = P.inf_norm(a) * (0.5 + 1e-3)
    assert float(sp.precond[0, 0]) == pytest.approx(1.0 / alpha, rel=1e-14)


@pytest.mark.parametrize("seed", range(4))
def test_construction_invariant_and_contraction(seed):
    import paper_2008_11480_b200 as P

    rng = np.random.default_rng(seed)
    a = _sdd(5, rng)
    for sp in (P.split_diagonal(a), P.split_scalar(a)):
        resid = np.eye(5) - _np(sp.precond) @ _np(sp.matrix)
        assert np.linalg.norm(resid - _np(sp.residual)) <= 1e-12 * np.linalg.norm(
            _np(sp.residual)) + 1e-14
        assert P.spectral_radius(sp.residual) < 1.0
    b = _spd(5, rng)
    for scale in (1e-6, 1e-3, 0.1):
        assert P.spectral_radius(P.split_scalar(b, eps=scale * P.inf_norm(b)).residual) < 1.0


def test_inconsistent_splitting_rejected():
    import paper_2008_11480_b200 as P

    with pytest.raises(ValueError):
        P.Splitting(precond=P.square_matrix([[0.5]]), residual=P.square_matrix([[0.7]]),
                    matrix=P.square_matrix([[2.0]]), kind="diagonal")


def test_two_s_minus_a_criterion():
    import paper_2008_11480_b200 as P

    assert P.check_two_s_minus_a(np.eye(3), P.split_diagonal(np.eye(3))) is True
    a = P.square_matrix([[2.0, 1.0], [1.0, 2.0]])
    assert P.check_two_s_minus_a(a, P.split_diagonal(a)) is True
    bad = P.Splitting(precond=P.square_matrix([[1.0]]), residual=P.square_matrix([[-3.0]]),
                      matrix=P.square_matrix([[4.0]]), kind="diagonal")
    assert P.check_two_s_minus_a(P.square_matrix([[4.0]]), bad) is False
    for seed in range(5):
        rng = np.random.default_rng(seed)
        a = _spd(4, rng)
        bad_alpha = float(np.min(np.linalg.eigvalsh(a))) / 4.0
        splits = [P.split_scalar(a), P.Splitting(
            precond=P.square_matrix(np.eye(4) / bad_alpha),
            residual=P.square_matrix(np.eye(4) - a / bad_alpha), matrix=P.square_matrix(a),
            kind="scalar")]
        for sp in splits:
            rho = P.spectral_radius(sp.residual, tol=1e-10)
            if abs(rho - 1.0) > 1e-6:
                assert P.check_two_s_minus_a(a, sp) == (rho < 1.0)


def test_positive_definite_and_rho_hint():
    import paper_2008_11480_b200 as P

    assert P.is_positive_definite(np.eye(3))
    assert not P.is_positive_definite(P.square_matrix([[1.0, 2.0], [2.0, 1.0]]))
    assert not P.is_positive_definite(np.zeros((2, 2)))
    assert not P.is_positive_definite(P.square_matrix([[1.0, 1.0], [1.0, 1.0 + 1e-16]]))
    sp = P.split_diagonal(_sdd(4, np.random.default_rng(7)))
    assert sp.rho_hint is None
    m = P.with_measured_rho(sp)
    assert m.rho_hint is not None and 0.0 <= m.rho_hint < 1.0
