"""Pin the CPU oracle against the reference's own outputs (tests/golden, made by
running the unmodified reference: tests/golden/make_golden.py)."""

import json
import os

import pytest

import cases
from conftest import GOLDEN


@pytest.fixture(scope="module")
def B():
    return cases.OracleBackend()


def test_plan_catalogue_matches_reference(B):
    with open(os.path.join(GOLDEN, "plans.json")) as fh:
        ref = json.load(fh)
    o = B.o
    for h, (s, cost, poly) in ref["plan_order"].items():
        node = o.plan_order(int(h))
        assert o.node_str(node) == s
        assert o.node_poly_cost(node) == poly and poly + 1 == cost
    for order, rows in ref["table"].items():
        mine = o.TABLE_ROOTS[int(order)]
        assert [lab for lab, _ in mine] == [r[0] for r in rows]
        for (lab, node), (_, s, cost, poly) in zip(mine, rows):
            assert o.node_str(node) == s and o.node_poly_cost(node) == poly
    s, cost, poly, ei = ref["order45"]
    assert o.node_str(o.order45()) == s and o.node_poly_cost(o.order45()) == poly


# The oracle performs the reference's numpy operations in the reference's
# order, so it reproduces the fixtures to the last bits (1e-13 allows for a
# different BLAS build on the GPU host).
@pytest.mark.parametrize("name,fixture", [
    ("toolkit", "toolkit.npz"), ("ns", "ns.npz"), ("richardson", "richardson.npz"),
    ("c1", "c1.npz"), ("c3", "c3.npz"), ("c4", "c4.npz"), ("c5", "c5.npz"),
])
def test_oracle_reproduces_reference(B, name, fixture):
    out = getattr(cases, f"case_{name}")(B)
    cases.compare(out, fixture, B, rtol=1e-12, ftol=1e-13)


def test_oracle_batched_fixture(B):
    cases.compare(cases.case_c2_oracle(B), "c2.npz", B, rtol=1e-12, ftol=1e-13)


def test_oracle_setup_path_matches_reference():
    """Symmetry check, PD verdicts (loop and blocked forms) and spectral radius
    of the oracle against the reference's outputs (setup.npz)."""
    import numpy as np

    from conftest import golden
    from oracle import seriesinv_oracle as O

    g = golden("setup.npz")
    for i in range(5):
        asym, fro, out = O.check_symmetric(g[f"sym{i}_a"])
        ok = int(asym <= 1e-10 * max(fro, 1e-300))
        assert ok == int(g[f"sym{i}_ok"])
        if ok:
            assert np.array_equal(out, g[f"sym{i}_out"])
    for i in range(int(g["pd_count"])):
        a = g[f"pd{i}_a"]
        assert int(O.is_positive_definite(a)) == int(g[f"pd{i}_default"]), i
        assert int(O.is_positive_definite(a, pivot_tol=0.0)) == int(g[f"pd{i}_zero_tol"]), i
        assert int(O.is_positive_definite_blocked(a, nb=32)) == int(g[f"pd{i}_default"]), i
    for i in range(int(g["rho_count"])):
        assert O.spectral_radius(g[f"rho{i}_a"]) == float(g[f"rho{i}"])
