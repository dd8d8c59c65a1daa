"""Series evaluators on the device: the behaviours the
reference's series-toolkit tests pin -- Horner conventions and counts, the
factored evaluator's count law and validation, every plan (order 2-64, the
table catalogue, order 45) equal to Horner with its advertised counts in both
modes, nested_eval with Y = 0 / malformed plans / the identity chain, and
geometric_apply incl. the doubling path."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _inst(seed, dim=5):
    """(x, y, a): x = S^-1, y = B of a scalar splitting of a random SPD a."""
    import paper_2008_11480_b200 as P

    rng = np.random.default_rng(seed)
    m = rng.standard_normal((dim, dim))
    a = P.square_matrix(m @ m.T / dim + 0.5 * np.eye(dim))
    sp = P.split_scalar(a)
    return sp.precond, sp.residual, a


def _rel(out, ref):
    return np.linalg.norm(_np(out) - _np(ref)) / max(np.linalg.norm(_np(ref)), 1e-300)


def test_horner_conventions():
    import paper_2008_11480_b200 as P

    x, y, a = _inst(0)
    ctr = P.MulCounter()
    assert torch.equal(P.horner_eval(y, x, 1, ctr), x) and ctr.mmm == 0
    xr = P.as_device(np.random.default_rng(1).standard_normal((3, 3)))
    for h in (1, 2, 7):
        assert torch.equal(P.horner_eval(P.as_device(np.zeros((3, 3))), xr, h, P.MulCounter()), xr)
    ctr = P.MulCounter()
    out = P.horner_eval(P.square_matrix([[0.5]]), P.square_matrix([[1.0]]), 4, ctr)
    assert float(out[0, 0]) == 1.875 and ctr.mmm == 3
    for h in (1, 2, 5, 11):
        c1, c2 = P.MulCounter(), P.MulCounter()
        P.horner_eval(y, x, h, c1)
        P.horner_eval(y, x, h, c2, a=a, form_y=True)
        assert (c1.mmm, c2.mmm) == (h - 1, h)
    with pytest.raises(ValueError):
        P.horner_eval(y, x, 0, P.MulCounter())
    for form_y in (False, True):
        with pytest.raises(ValueError):
            P.horner_eval(None, x, 3, P.MulCounter(), form_y=form_y)


def test_factored_evaluator():
    import paper_2008_11480_b200 as P

    x, y, a = _inst(2)
    ctr = P.MulCounter()
    assert torch.equal(P.factored_eval(y, x, a, 0, 1, ctr), x) and ctr.mmm == 1
    ctr = P.MulCounter()
    out = P.factored_eval(y, x, a, 8, 5, ctr)
    assert ctr.mmm == 14 and _rel(out, P.horner_eval(y, x, 45, P.MulCounter())) <= 1e-10
    x4, y4, a4 = _inst(3, dim=4)
    assert _rel(P.factored_eval(y4, x4, a4, 2, 3, P.MulCounter()),
                P.horner_eval(y4, x4, 9, P.MulCounter())) <= 1e-10
    for p in range(8):
        for w in range(1, 7):
            ctr = P.MulCounter()
            P.factored_eval(y4, x4, a4, p, w, ctr)
            expected = p + 1 if w == 1 else (w if p == 0 else p + w + 1)
            assert ctr.mmm == expected == P.factored_mmm(p, w)
    for p, w, poly in ((2, 3, 5), (3, 1, 3), (0, 4, 3), (5, 2, 7)):
        ctr = P.MulCounter()
        P.factored_eval(y4, x4, a4, p, w, ctr, form_y=False)
        assert ctr.mmm == poly == P.factored_mmm(p, w) - 1
    with pytest.raises(ValueError):
        P.factored_eval(y + 0.5, x, a, 1, 2, P.MulCounter())
    for p, w in ((-1, 2), (2, 0)):
        with pytest.raises(ValueError):
            P.factored_eval(y, x, a, p, w, P.MulCounter())


def test_every_plan_matches_horner_with_its_counts():
    import paper_2008_11480_b200 as P

    x, y, a = _inst(4, dim=4)
    refs = {}
    plans = [(f"h{h}", h, P.plan_order(h)) for h in range(2, 65)]
    plans += [(lab, order, plan) for order, ps in P.table_plans().items()
              for lab, plan in zip(P.TABLE_LABELS[order], ps)]
    plans.append(("order45", 45, P.order45_plan()))
    for label, order, plan in plans:
        if order not in refs:
            refs[order] = P.horner_eval(y, x, order, P.MulCounter())
        c1, c2 = P.MulCounter(), P.MulCounter()
        out = P.nested_eval(y, x, a, plan, c1)
        P.nested_eval(y, x, a, plan, c2, form_y=False)
        assert _rel(out, refs[order]) <= 1e-8, label
        assert (c1.mmm, c2.mmm) == (plan.mmm_cost, plan.mmm_poly), label


def test_nested_eval_edges_and_identity_chain():
    import paper_2008_11480_b200 as P

    a2 = P.square_matrix(np.eye(3) * 2.0)
    xh = P.square_matrix(np.eye(3) * 0.5)
    for plan in (P.order45_plan(), P.plan_order(7), P.table_plans()[8][0]):
        assert np.allclose(_np(P.nested_eval(None, xh, a2, plan, P.MulCounter())), _np(xh),
                           atol=1e-15)
    x, y, a = _inst(5)
    bogus = P.FactorPlan(order_h=5, root=P.Horner(4), mmm_cost=4, mmm_poly=3,
                         efficiency_index=1.0)
    with pytest.raises(ValueError):
        P.nested_eval(y, x, a, bogus, P.MulCounter())
    x4, y4, a4 = _inst(6, dim=4)
    for plan in (P.plan_order(6), P.plan_order(12), P.order45_plan()):
        z = P.nested_eval(y4, x4, a4, plan, P.MulCounter())
        lhs = np.eye(4) - _np(z) @ _np(a4)
        target = np.linalg.matrix_power(_np(y4), plan.order_h)
        assert np.linalg.norm(lhs - target) <= 1e-8 * max(np.linalg.norm(target), 1e-300)


@pytest.mark.parametrize("order", [1, 2, 3, 19, 20, 64, 65, 130, 200])
def test_geometric_apply(order):
    import paper_2008_11480_b200 as P

    x, y, a = _inst(7 + order, dim=4)
    out = P.geometric_apply(y, x, order, a, P.MulCounter())
    assert _rel(out, P.horner_eval(y, x, order, P.MulCounter())) <= 1e-9
    with pytest.raises(ValueError):
        P.geometric_apply(y, x, 0, a, P.MulCounter())
