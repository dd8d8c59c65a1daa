"""Host-side integer laws and argument validation of the product package (no GPU)."""

import pytest

import paper_2008_11480_b200 as P


def test_exponent_laws_examples():
    assert P.residual_exponent("classical", 2, 3, 1) == 9
    assert P.residual_exponent("double", 1, 2, 1) == 6
    assert P.residual_exponent("double", 3, 2, 2) == 112
    assert P.residual_exponent("composite", 1, 2, 1, rates=(2, 3)) == 7
    assert P.residual_exponent("additive", 2, 3, 1) == 13
    assert P.additive_exponents(2, 3, 1) == (9, 13)
    with pytest.raises(ValueError):
        P.residual_exponent("composite", 1, 2, 1)
    with pytest.raises(ValueError):
        P.residual_exponent("mystery", 1, 2, 1)


def test_double_law_recursion():
    for n in range(2, 7):
        for h in range(1, 5):
            e = h
            for k in range(1, 9):
                e = n * (h * n**k) + n * e
                assert e == P.double_exponent(k, n, h)


def test_richardson_closed_forms():
    assert P.step_exponent_qn(1, 2, 1) == 16
    assert P.step_exponent_general(1, 2, 1, 3) == 22
    for n in range(2, 7):
        for h in range(1, 5):
            for k in range(1, 13):
                assert P.cumulative_exponent_closed(k, n, h) == P.cumulative_exponent(k, n, h)
    tm = P.transient_model(3, 2, 1, rho=0.5, theta0_norm=2.0)
    assert tm.total_exponent == 192 and tm.step_exponent == 128
    assert tm.bound == pytest.approx(2.0 * 0.5**192)
    with pytest.raises(ValueError):
        P.cumulative_exponent_closed(3, 1, 1)


def test_composite_spec_validation():
    with pytest.raises(ValueError):
        P.CompositeSpec(())
    with pytest.raises(ValueError):
        P.CompositeSpec((0, 2))
    assert P.constant_rates(3, 2).rates == (3, 3)
    stepper = P.power_rates(2, 3)
    assert stepper(0).rates == (1, 1, 1) and stepper(3).rates == (8, 8, 8)
    with pytest.raises(ValueError):
        P.power_rates(1, 2)


def test_counter_semantics():
    c = P.MulCounter(2, 1)
    c.merge(P.MulCounter(3, 4))
    assert (c.mmm, c.mvm) == (5, 5)
    with pytest.raises(ValueError):
        c.count_mmm(-1)
    buf = [7, 2]
    c.absorb(buf)
    assert (c.mmm, c.mvm) == (12, 7)


def test_peer_gather_agreement_check():
    """SI_PEER_CHECK's divergence check (peer.py): ranks that pair a gather
    with different (slot, epoch) fail loudly."""
    import types

    import pytest

    from paper_2008_11480_b200.peer import PeerComm

    fabric = types.SimpleNamespace()  # stands in for the virtual ranks' shared fabric

    def rank(r):
        c = PeerComm.__new__(PeerComm)
        c.rank, c.world, c.fabric, c.seq = r, 2, types.SimpleNamespace(fabric=fabric), 1
        return c

    rank(0)._check_agreement(3, 7, 64)
    rank(1)._check_agreement(3, 7, 64)  # same pairing: fine
    a, b = rank(0), rank(1)
    a.seq = b.seq = 2
    a._check_agreement(1, 4, 64)
    with pytest.raises(RuntimeError, match="diverged"):
        b._check_agreement(2, 4, 64)
