"""matrix_core on the device (matrix_core.py:52-239): the
behaviours the reference's matrix-core tests pin -- construction checks,
products (identity, diagonal, dot-product error bound, dimension errors,
counters), powers, associativity, the power iteration (incl. paired and
complex dominant eigenvalues) and the norms."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def test_construction_checks():
    import paper_2008_11480_b200 as P

    with pytest.raises(ValueError):
        P.square_matrix([[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]])
    with pytest.raises(ValueError):
        P.square_matrix([[1.0, np.nan], [0.0, 1.0]])
    with pytest.raises(ValueError):
        P.vector([np.inf, 1.0])


def test_products_and_counters():
    import paper_2008_11480_b200 as P

    rng = np.random.default_rng(1)
    m = rng.standard_normal((3, 3))
    ctr = P.MulCounter()
    assert np.array_equal(_np(P.mat_mul(np.eye(3), m, ctr)), m) and ctr.mmm == 1
    assert np.array_equal(_np(P.mat_mul(np.diag([2.0, 3.0]), np.diag([5.0, 7.0]), ctr)),
                          np.diag([10.0, 21.0]))
    a, b = rng.standard_normal((4, 4)), rng.standard_normal((4, 4))
    naive = np.array([[sum(a[i, k] * b[k, j] for k in range(4)) for j in range(4)]
                      for i in range(4)])
    assert np.allclose(_np(P.mat_mul(a, b, P.MulCounter())), naive, rtol=0, atol=1e-13)
    with pytest.raises(ValueError):
        P.mat_mul(np.eye(2), np.eye(3), P.MulCounter())
    with pytest.raises(ValueError):
        P.mat_vec(np.eye(2), np.zeros(3), P.MulCounter())
    ctr = P.MulCounter()
    for _ in range(5):
        P.mat_mul(m, m, ctr)
    P.mat_vec(m, np.zeros(3), ctr)
    assert (ctr.mmm, ctr.mvm) == (5, 1)
    c1, c2 = P.MulCounter(2, 1), P.MulCounter(3, 4)
    c1.merge(c2)
    assert (c1.mmm, c1.mvm) == (5, 5)


@pytest.mark.parametrize("e1,e2", [(0, 5), (1, 1), (7, 13), (31, 64), (64, 64)])
def test_powers(e1, e2):
    import paper_2008_11480_b200 as P

    rng = np.random.default_rng(e1 * 100 + e2)
    m = rng.standard_normal((4, 4))
    m = 0.9 * m / np.linalg.norm(m, 2)
    assert np.array_equal(_np(P.mat_pow(m, 0)), np.eye(4))
    assert np.array_equal(_np(P.mat_pow(m, 1)), m)
    lhs = _np(P.mat_pow(m, e1 + e2))
    rhs = _np(P.mat_mul(P.mat_pow(m, e1), P.mat_pow(m, e2), P.MulCounter()))
    assert np.linalg.norm(lhs - rhs) <= 1e-11 * max(np.linalg.norm(lhs), 1e-300)
    assert np.allclose(np.diag(_np(P.mat_pow(np.diag([0.5, 0.2]), 6))), [0.015625, 0.000064],
                       rtol=1e-12)
    with pytest.raises(ValueError):
        P.mat_pow(np.eye(2), -1)
    ctr = P.MulCounter()
    assert np.allclose(_np(P.mat_pow_counted(m, 6, ctr)), _np(P.mat_pow(m, 6)), rtol=1e-12,
                       atol=1e-15)
    assert ctr.mmm > 0
    assert np.array_equal(_np(P.mat_pow_counted(m, 0, P.MulCounter())), np.eye(4))


@pytest.mark.parametrize("dim,seed", [(2, 0), (5, 1), (8, 2), (3, 99)])
def test_associativity_and_counter_determinism(dim, seed):
    import paper_2008_11480_b200 as P

    r = np.random.default_rng(seed)
    a, b, c = (r.standard_normal((dim, dim)) for _ in range(3))
    ctr = P.MulCounter()
    left = _np(P.mat_mul(P.mat_mul(a, b, ctr), c, ctr))
    right = _np(P.mat_mul(a, P.mat_mul(b, c, ctr), ctr))
    bound = 1e-12 * np.linalg.norm(a) * np.linalg.norm(b) * np.linalg.norm(c)
    assert np.linalg.norm(left - right) <= bound

    def work():
        k = P.MulCounter()
        mm = P.mat_mul(a, a, k)
        P.mat_pow_counted(mm, 9, k)
        P.mat_vec(mm, np.ones(dim), k)
        return k.mmm, k.mvm

    assert work() == work()


def test_spectral_radius_cases():
    import paper_2008_11480_b200 as P

    assert P.spectral_radius(np.diag([0.9, 0.1])) == pytest.approx(0.9, rel=1e-10)
    assert P.spectral_radius(np.eye(4)) == pytest.approx(1.0, rel=1e-12)
    assert P.spectral_radius(np.zeros((3, 3))) == 0.0
    assert P.spectral_radius(np.array([[0.0, -0.5], [-0.5, 0.0]])) == pytest.approx(0.5,
                                                                                     rel=1e-10)
    for seed in range(6):
        m = np.random.default_rng(seed).standard_normal((5, 5))
        sym = (m + m.T) / 2.0
        expected = float(np.max(np.abs(np.linalg.eigvalsh(sym))))
        assert P.spectral_radius(sym) == pytest.approx(expected, rel=1e-8)
    with pytest.raises(P.SpectralRadiusError) as err:   # complex dominant pair
        P.spectral_radius(np.array([[0.0, 2.0], [-0.5, 0.0]]), max_iter=300)
    assert 0.0 < err.value.best_estimate <= 2.0


def test_norms():
    import paper_2008_11480_b200 as P

    assert P.norms(np.array([[1.0, -2.0], [3.0, 4.0]])).inf_norm == 7.0
    for n in (1, 3, 7):
        assert P.norms(np.eye(n)).frobenius == pytest.approx(np.sqrt(n), rel=1e-15)
    assert tuple(P.norms(np.zeros((4, 4)))) == (0.0, 0.0)
    assert P.fro_norm(np.zeros((2, 2))) == 0.0 and P.inf_norm(np.zeros((2, 2))) == 0.0
