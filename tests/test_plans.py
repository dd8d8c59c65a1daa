"""Host-side plan logic of the product package vs the reference catalogue
(tests/golden/plans.json, recorded from the reference) -- no GPU needed."""

import json
import os

import pytest

import paper_2008_11480_b200.series_toolkit as st
from conftest import GOLDEN

with open(os.path.join(GOLDEN, "plans.json")) as fh:
    REF = json.load(fh)


@pytest.mark.parametrize("h", range(2, 65))
def test_plan_order_matches_reference(h):
    s, cost, poly = REF["plan_order"][str(h)]
    p = st.plan_order(h)
    assert st.plan_str(p) == s
    assert (p.mmm_cost, p.mmm_poly, p.order_h) == (cost, poly, h)


def test_table_plans_match_reference():
    plans = st.table_plans()
    assert sorted(plans) == sorted(int(k) for k in REF["table"])
    for order, rows in REF["table"].items():
        mine = plans[int(order)]
        assert list(st.TABLE_LABELS[int(order)]) == [r[0] for r in rows]
        for p, (_, s, cost, poly) in zip(mine, rows):
            assert (st.plan_str(p), p.mmm_cost, p.mmm_poly) == (s, cost, poly)


def test_order45():
    s, cost, poly, ei = REF["order45"]
    p = st.order45_plan()
    assert (st.plan_str(p), p.mmm_cost, p.mmm_poly) == (s, cost, poly)
    assert p.efficiency_index == pytest.approx(ei, rel=1e-14)
    assert p.efficiency_index == pytest.approx(1.4633, abs=5e-5)


def test_cost_model():
    assert st.factored_mmm(8, 5) == 14 and st.factored_mmm(3, 1) == 4 and st.factored_mmm(0, 4) == 4
    assert st.efficiency_index(1, 1) == pytest.approx(2 ** 0.5)
    assert st.split_candidates(18) == [(1, 9), (2, 6), (5, 3), (8, 2)]
    with pytest.raises(ValueError):
        st.factored_mmm(-1, 2)


def test_plan_validation():
    with pytest.raises(ValueError):
        st.plan_order(1)
    with pytest.raises(ValueError):
        st.plan_order(65)
    with pytest.raises(ValueError):
        st.make_plan(st.Split(2, 2, st.Horner(2), st.Horner(2)))  # inner order != p+1
    with pytest.raises(ValueError):
        st.make_plan(st.Split(1, 3, st.Horner(2), None))  # missing outer
    with pytest.raises(ValueError):
        st.make_plan(st.Horner(0))


def _decode(code, consts):
    """Python decoder of the int32 preorder code (mirror of engine.cu Decoder)."""
    pos = 0

    def nxt():
        nonlocal pos
        pos += 1
        return code[pos - 1]

    def node():
        kind = nxt()
        if kind == 0:
            return st.Horner(nxt())
        if kind == 1:
            p, w = nxt(), nxt()
            inner = node() if nxt() else None
            outer = node() if nxt() else None
            return st.Split(p, w, inner, outer)
        if kind == 2:
            return st.PrimeWrap(node())
        order, nregs, ninstr = nxt(), nxt(), nxt()
        prog = []
        for _ in range(ninstr):
            op, dst = nxt(), nxt()
            if op == 0:
                prog.append(("mul", dst, nxt(), nxt()))
            elif op == 1:
                prog.append(("res", dst, nxt()))
            else:
                c = consts[nxt()]
                nt = nxt()
                prog.append(("lin", dst, c, tuple((consts[nxt()], nxt()) for _ in range(nt))))
        return ("table", order, nregs, tuple(prog))

    n = node()
    assert pos == len(code)
    return n


@pytest.mark.parametrize("h", [2, 3, 5, 8, 16, 45, 64])
def test_encoding_roundtrip_structure(h):
    plan = st.order45_plan() if h == 45 else st.plan_order(h)
    code, consts = st.encode_plan(plan)
    dec = _decode(code, consts)

    def order(n):
        if isinstance(n, tuple):
            return n[1]
        if isinstance(n, st.Horner):
            return n.order
        if isinstance(n, st.Split):
            if n.p >= 1:
                assert order(n.inner) == n.p + 1
            if n.w >= 2:
                assert order(n.outer) == n.w
            return n.w * (n.p + 1)
        return order(n.inner) + 1

    assert order(dec) == h


def test_table_form_register_encoding():
    code, consts = st.encode_plan(st.table_plans()[8][0])
    dec = _decode(code, consts)
    kind, order, nregs, prog = dec
    assert order == 8 and nregs == 2 + 8  # Y, X + c0 c1 q2 c2 c3 q4 c4 z
    assert [p[0] for p in prog] == ["mul", "lin", "res", "mul", "lin", "res", "mul", "lin"]
    assert prog[0] == ("mul", 2, 0, 1)  # c0 = Y X
    assert prog[1] == ("lin", 3, 0.0, ((1.0, 1), (1.0, 2)))  # c1 = X + c0


def test_geometric_base_orders():
    assert st.geometric_base_order(64) == 64
    assert st.geometric_base_order(65) == 32
    assert st.geometric_base_order(200) == 50
    assert st.geometric_base_plan(1) is None
