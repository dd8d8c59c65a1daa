"""Richardson steps on the device: the behaviours the
reference's Richardson tests pin -- the mismatch contraction law
theta_k - theta* = B^gamma_k (theta_0 - theta*), q != n, the recursive form
matching the direct form with fewer products from the second step, the
carried weight, exact cases, executor bitwise equality, and acceleration over
the plain estimator."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _contractive(dim, rho, rng):
    """(A, eps): scalar splitting with alpha = 1 and symmetric B, rho(B) = rho."""
    for _ in range(100):
        q, _ = np.linalg.qr(rng.standard_normal((dim, dim)))
        eig = rng.uniform(-0.6 * rho, 0.6 * rho, dim)
        eig[0] = rho
        b = (q * eig) @ q.T
        a = np.eye(dim) - (b + b.T) / 2.0
        eps = 1.0 - np.abs(a).sum(axis=1).max() / 2.0
        if eps > 1e-6:
            return a, float(eps)
    raise RuntimeError("no contractive system")


def _setup(dim, rho, seed):
    import paper_2008_11480_b200 as P

    rng = np.random.default_rng(seed)
    a, eps = _contractive(dim, rho, rng)
    sp = P.split_scalar(a, eps)
    theta_star = rng.standard_normal(dim)
    return P.square_matrix(a), sp, theta_star, P.as_device(a @ theta_star)


def _law(st, sp, theta_star, t0, gamma, rel):
    target = np.linalg.matrix_power(_np(sp.residual), gamma) @ t0
    err = _np(st.theta) - theta_star
    if np.linalg.norm(target) < 1e-250:
        assert np.linalg.norm(err) <= 1e-200
    else:
        assert np.linalg.norm(err - target) <= rel * np.linalg.norm(target)


def test_direct_step_laws():
    import paper_2008_11480_b200 as P

    a = P.square_matrix(np.eye(3))
    ts = np.array([1.0, -2.0, 0.5])
    st = P.initial_richardson(P.split_scalar(a, eps=0.5), P.as_device(ts))
    assert np.allclose(_np(st.theta), ts, atol=1e-15)
    a, sp, ts, b = _setup(4, 0.98, 0)
    st = P.initial_richardson(sp, b, order=2, q=2)
    t0 = _np(st.theta) - ts
    st = P.richardson_step(st, a, b)
    _law(st, sp, ts, t0, 16, 1e-9)
    rho = float(np.max(np.abs(np.linalg.eigvalsh(_np(sp.residual)))))
    assert np.linalg.norm(_np(st.theta) - ts) <= rho ** 16 * np.linalg.norm(t0) * (1 + 1e-6)
    st = P.initial_richardson(sp, b, order=2, q=3)
    t0 = _np(st.theta) - ts
    _law(P.richardson_step(st, a, b), sp, ts, t0, 22, 1e-9)


@pytest.mark.parametrize("n,h,pw", [(2, 1, (0, 1)), (2, 2, (1, 1)), (3, 1, (0, 1)), (3, 2, (1, 1))])
def test_mismatch_model(n, h, pw):
    import paper_2008_11480_b200 as P

    a, sp, ts, b = _setup(5, 0.999, 10 * n + h)
    st = P.initial_richardson(sp, b, pw[0], pw[1], order=n, q=n)
    t0 = _np(st.theta) - ts
    for k in range(1, 4):
        st = P.richardson_step(st, a, b)
        _law(st, sp, ts, t0, P.cumulative_exponent(k, n, h), 1e-8)
    # A^-1 (b - A theta_k) = theta* - theta_k
    rec = np.linalg.solve(_np(a), _np(b) - _np(a) @ _np(st.theta))
    mis = _np(st.theta) - ts
    assert np.linalg.norm(rec + mis) <= 1e-8 * max(np.linalg.norm(mis), 1e-300)


def test_recursive_step_behaviour():
    import paper_2008_11480_b200 as P

    a, sp, ts, b = _setup(4, 0.9, 1)
    with pytest.raises(ValueError):
        P.richardson_recursive_step(P.initial_richardson(sp, b, order=2, q=3), a, b)
    for n in (2, 3):
        a, sp, ts, b = _setup(5, 0.995, 2 + n)
        direct = P.initial_richardson(sp, b, 1, 2, order=n, q=n)
        recur = P.initial_richardson(sp, b, 1, 2, order=n, q=n)
        for _ in range(4):
            direct = P.richardson_step(direct, a, b)
            recur = P.richardson_recursive_step(recur, a, b)
            assert np.linalg.norm(_np(recur.theta) - _np(direct.theta)) <= 1e-9 * max(
                np.linalg.norm(_np(direct.theta)), 1e-300)
    a, sp, ts, b = _setup(4, 0.99, 6)
    st = P.initial_richardson(sp, b, order=2, q=2)
    for _ in range(3):
        st = P.richardson_recursive_step(st, a, b)
        inner = st.inner
        sum_fg = P.horner_eval(inner.residual, inner.estimate, st.q, P.MulCounter())
        weight = _np(inner.accel_estimate) + _np(inner.accel_residual) @ _np(sum_fg)
        assert np.linalg.norm(_np(st.omega) - weight) <= 1e-9 * np.linalg.norm(_np(st.omega))
    for n in (2, 3, 4):
        a, sp, ts, b = _setup(4, 0.95, 7 + n)
        direct = P.initial_richardson(sp, b, order=n, q=n)
        recur = P.initial_richardson(sp, b, order=n, q=n)
        for k in range(1, 5):
            d0, r0 = direct.ctr.mmm, recur.ctr.mmm
            direct = P.richardson_step(direct, a, b)
            recur = P.richardson_recursive_step(recur, a, b)
            dc, rc = direct.ctr.mmm - d0, recur.ctr.mmm - r0
            assert rc == dc if k == 1 else rc < dc
    a = P.square_matrix(np.eye(3))
    ts = np.array([2.0, 0.0, -1.0])
    st = P.initial_richardson(P.split_scalar(a, eps=0.5), P.as_device(ts))
    st = P.richardson_recursive_step(st, a, P.as_device(ts))
    assert np.allclose(_np(st.theta), ts, atol=1e-14)
    assert np.linalg.norm(_np(st.omega) - np.eye(3)) <= 1e-12


def test_recursive_executor_bitwise_and_acceleration():
    import paper_2008_11480_b200 as P

    a, sp, ts, b = _setup(5, 0.99, 20)
    serial = P.initial_richardson(sp, b, 1, 2, order=2, q=2)
    threaded = P.initial_richardson(sp, b, 1, 2, order=2, q=2)
    with ThreadPoolExecutor(max_workers=2) as pool:
        for _ in range(3):
            serial = P.richardson_recursive_step(serial, a, b)
            threaded = P.richardson_recursive_step(threaded, a, b, executor=pool)
    assert torch.equal(serial.theta, threaded.theta) and torch.equal(serial.omega, threaded.omega)
    assert serial.ctr.mmm == threaded.ctr.mmm
    rich = P.initial_richardson(sp, b, order=2, q=2)
    plain = P.initial_series(sp, 0, 1, order=2)
    for _ in range(3):
        rich = P.richardson_step(rich, a, b)
        plain = P.ns_step(plain, a)
    theta_plain = P.mat_vec(plain.estimate, b, plain.ctr)
    assert np.linalg.norm(_np(rich.theta) - ts) <= np.linalg.norm(_np(theta_plain) - ts)


@pytest.mark.parametrize("backend,concurrent,factorised", [
    ("dmma", False, False), ("dmma", True, True), ("ozaki", False, True)])
def test_recursive_step_with_copies_in_flight(backend, concurrent, factorised):
    """si_richardson_recursive_step_ex: every input copied host->device on another
    stream behind its own event, every field of the new state read back behind
    the event the step records for it -- bitwise the plain call (first call and
    steady state), same product counts."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    n, rhs = 1024, 4
    a, _ = configs.c3_gram(n=n, shift=1e-3)
    b = np.random.default_rng(5).standard_normal((n, rhs))
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    bd = P.as_device(b)
    kw = dict(factor_plan=P.plan_order(16), doubling_sum=True) if factorised else {}
    ex = True if concurrent else None
    names = {"a": "a", "b": "b", "theta": "theta", "g": "estimate", "f": "residual",
             "l": "accel_estimate", "r": "accel_residual", "omega": "omega", "ns": "ns_part"}

    def fields(st):
        return {"theta": st.theta, "g": st.inner.estimate, "f": st.inner.residual,
                "l": st.inner.accel_estimate, "r": st.inner.accel_residual,
                "omega": st.omega, "ns": st.ns_part}

    def in_flight(st):
        host = {k: v.cpu().pin_memory() for k, v in fields(st).items() if v is not None}
        host["a"], host["b"] = sp.matrix.cpu().pin_memory(), bd.cpu().pin_memory()
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        main = torch.cuda.current_stream()
        up.wait_stream(main)
        d, ready = {}, {}
        with torch.cuda.stream(up):
            torch.cuda._sleep(20_000_000)  # the step must wait, not race
            for k in ("f", "g", "ns", "omega", "theta", "b", "a", "l", "r"):
                if k not in host:
                    continue
                d[k] = host[k].to("cuda", non_blocking=True)
                d[k].record_stream(main)
                ready[names[k]] = torch.cuda.Event()
                ready[names[k]].record(up)
        inner = P.DoubleNsState(estimate=d["g"], residual=d["f"], accel_estimate=d["l"],
                                accel_residual=d["r"], step=st.inner.step, order=16,
                                series_order=st.inner.series_order, ctr=P.MulCounter())
        st2 = P.RichardsonState(theta=d["theta"], inner=inner, q=16, omega=d.get("omega"),
                                ns_part=d.get("ns"), step=st.step, ctr=inner.ctr)
        outs = ("accel_estimate", "accel_residual", "estimate", "residual", "ns_part", "omega",
                "theta")
        done = {k: torch.cuda.Event() for k in outs}
        new = P.richardson_recursive_step(st2, d["a"], d["b"], executor=ex, inputs_ready=ready,
                                          outputs_done=done, **kw)
        back = {}
        rev = {v: k for k, v in names.items()}
        for k in outs:
            v = fields(new)[rev[k]]
            down.wait_event(done[k])
            v.record_stream(down)
            with torch.cuda.stream(down):
                back[rev[k]] = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
                back[rev[k]].copy_(v, non_blocking=True)
        down.synchronize()
        return new, back

    with P.gemm_backend(backend, moduli=16, min_dim=1024) if backend == "ozaki" \
            else P.gemm_backend("dmma"):
        st = P.initial_richardson(sp, bd, order=16, q=16)
        for _ in range(2):  # the first call (no omega / ns_part yet), then the steady state
            before = st.ctr.mmm
            ref = P.richardson_recursive_step(st, sp.matrix, bd, executor=ex, **kw)
            new, back = in_flight(st)
            torch.cuda.synchronize()
            for k, v in fields(ref).items():
                assert torch.equal(v, fields(new)[k]), k
                assert torch.equal(v.cpu(), back[k]), k
            assert new.ctr.mmm == ref.ctr.mmm - before
            st = ref
    with pytest.raises(ValueError):
        P.richardson_recursive_step(st, sp.matrix, bd, inputs_ready={"bogus": None})
