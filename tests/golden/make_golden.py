"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED reference.

Run in the build container (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``seriesinv`` from /root/reference/pkg/src, feeds it seeded inputs
(shapes and recipes of BASELINE.json's configs at reduced sizes, plus small
instances of every hot-path function) and stores inputs, outputs and
MulCounter deltas.  The fixtures pin the oracle (tests/test_oracle_golden.py)
and the CUDA path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = os.environ.get("SERIESINV_REF", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import seriesinv as si  # noqa: E402  (the reference)

from paper_2008_11480_b200 import configs  # noqa: E402  (host generators only)


def spd(dim, rng, shift=0.5):
    m = rng.standard_normal((dim, dim))
    return m @ m.T / dim + shift * np.eye(dim)


def sdd_balanced(dim, rho, rng, jitter=0.002):
    """Symmetric SDD matrix whose diagonal splitting has rho(B) ~= rho."""
    w = rng.uniform(0.5, 1.5, (dim, dim))
    w = (w + w.T) / 2.0
    np.fill_diagonal(w, 0.0)
    for _ in range(200):
        s = np.sqrt(w.sum(axis=1) / rho)
        w = w / np.outer(s, s)
    return np.diag(1.0 + jitter * rng.uniform(0.0, 1.0, dim)) - w


def contractive(dim, rho, rng):
    """(A, eps) whose scalar splitting has alpha = 1 and a symmetric B, rho(B) = rho."""
    for _ in range(100):
        q, _ = np.linalg.qr(rng.standard_normal((dim, dim)))
        eig = rng.uniform(-0.6 * rho, 0.6 * rho, dim)
        eig[0] = rho
        b = (q * eig) @ q.T
        a = np.eye(dim) - (b + b.T) / 2.0
        eps = 1.0 - si.inf_norm(a) / 2.0
        if eps > 1e-6:
            return a, float(eps)
    raise RuntimeError("no contractive system")


def plans_json():
    out = {"plan_order": {}, "table": {}, "order45": None}
    for h in range(2, 65):
        p = si.plan_order(h)
        out["plan_order"][h] = [si.plan_str(p), p.mmm_cost, p.mmm_poly]
    for order, plans in si.table_plans().items():
        out["table"][order] = [[lab, si.plan_str(p), p.mmm_cost, p.mmm_poly]
                               for lab, p in zip(si.series_toolkit.TABLE_LABELS[order], plans)]
    p = si.order45_plan()
    out["order45"] = [si.plan_str(p), p.mmm_cost, p.mmm_poly, p.efficiency_index]
    with open(os.path.join(HERE, "plans.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def toolkit():
    rng = np.random.default_rng(101)
    a = spd(6, rng)
    sp = si.split_scalar(a)
    x, y = sp.precond, sp.residual
    d = {"a": sp.matrix, "x": x, "y": y}
    for h in (1, 2, 3, 8):
        c = si.MulCounter()
        d[f"horner_{h}"] = si.horner_eval(y, x, h, c)
        d[f"horner_{h}_mmm"] = c.mmm
        c = si.MulCounter()
        d[f"hornerf_{h}"] = si.horner_eval(y, x, h, c, a=sp.matrix, form_y=True)
        d[f"hornerf_{h}_mmm"] = c.mmm
    for p, w in ((0, 1), (1, 1), (1, 2), (2, 3), (3, 4), (0, 3)):
        for fy in (True, False):
            c = si.MulCounter()
            d[f"factored_{p}_{w}_{int(fy)}"] = si.factored_eval(y, x, sp.matrix, p, w, c, form_y=fy)
            d[f"factored_{p}_{w}_{int(fy)}_mmm"] = c.mmm
    for h in range(2, 65):
        c = si.MulCounter()
        d[f"plan_{h}"] = si.nested_eval(y, x, sp.matrix, si.plan_order(h), c)
        d[f"plan_{h}_mmm"] = c.mmm
    for order, plans in si.table_plans().items():
        for lab, p in zip(si.series_toolkit.TABLE_LABELS[order], plans):
            c = si.MulCounter()
            d[f"table_{lab}"] = si.nested_eval(y, x, sp.matrix, p, c, form_y=False)
            d[f"table_{lab}_mmm"] = c.mmm
    c = si.MulCounter()
    d["order45"] = si.nested_eval(y, x, sp.matrix, si.order45_plan(), c)
    d["order45_mmm"] = c.mmm
    for order in (1, 2, 3, 19, 20, 64, 65, 130, 200):
        c = si.MulCounter()
        d[f"geom_{order}"] = si.geometric_apply(y, x, order, sp.matrix, c)
        d[f"geom_{order}_mmm"] = c.mmm
    for e in (0, 1, 5, 6, 13):
        c = si.MulCounter()
        d[f"pow_{e}"] = si.mat_pow_counted(y, e, c)
        d[f"pow_{e}_mmm"] = c.mmm
    m1 = rng.standard_normal((7, 5))
    m2 = rng.standard_normal((5, 3))
    d["mm_a"], d["mm_b"], d["mm_ab"] = m1, m2, si.mat_mul(m1, m2, si.MulCounter())
    np.savez_compressed(os.path.join(HERE, "toolkit.npz"), **d)


def ns_family():
    rng = np.random.default_rng(102)
    a = sdd_balanced(5, 0.95, rng)
    sp = si.split_diagonal(a)
    d = {"a": sp.matrix, "precond": sp.precond, "residual": sp.residual}
    for p, w, n in ((0, 1, 2), (1, 1, 3), (1, 2, 2), (2, 3, 4)):
        st = si.initial_series(sp, p, w, order=n)
        key = f"init_{p}_{w}"
        d[key + "_g"], d[key + "_f"], d[key + "_mmm"] = st.estimate, st.residual, st.ctr.mmm
        for k in range(3):
            st = si.ns_step(st, sp.matrix)
            d[f"ns_{p}_{w}_{n}_{k}_g"] = st.estimate
            d[f"ns_{p}_{w}_{n}_{k}_f"] = st.residual
            d[f"ns_{p}_{w}_{n}_{k}_mmm"] = st.ctr.mmm
    st = si.initial_series(sp, 0, 1, order=8)
    for k in range(2):
        st = si.ns_step(st, sp.matrix, plan=si.table_plans()[8][0])
        d[f"nsh8_{k}_g"], d[f"nsh8_{k}_f"], d[f"nsh8_{k}_mmm"] = st.estimate, st.residual, st.ctr.mmm
    for tag, rates, n in (("c23", (2, 3), 2), ("c2345", (2, 3, 4, 5), 2), ("c1", (1,), 1),
                          ("c100", (100,), 2), ("c22", (2, 2), 3)):
        st = si.initial_series(sp, 0, 1, order=n)
        for k in range(2):
            st = si.composite_step(st, sp.matrix, sp, si.CompositeSpec(rates), order_n=n)
            d[f"comp_{tag}_{k}_g"], d[f"comp_{tag}_{k}_f"] = st.estimate, st.residual
            d[f"comp_{tag}_{k}_mmm"] = st.ctr.mmm
    dst = si.initial_double(sp, 1, 2, order=3)
    d["dbl_init_g"], d["dbl_init_f"] = dst.estimate, dst.residual
    d["dbl_init_l"], d["dbl_init_r"], d["dbl_init_mmm"] = dst.accel_estimate, dst.accel_residual, dst.ctr.mmm
    for k in range(3):
        dst = si.double_ns_step(dst, sp.matrix)
        for f, v in (("g", dst.estimate), ("f", dst.residual), ("l", dst.accel_estimate),
                     ("r", dst.accel_residual)):
            d[f"dbl_{k}_{f}"] = v
        d[f"dbl_{k}_mmm"] = dst.ctr.mmm
    z = g = sp.precond
    ctr = si.MulCounter()
    for k in range(2):
        z, g = si.additive_correction_step(z, g, sp.matrix, 3, ctr)
        d[f"add_{k}_z"], d[f"add_{k}_g"], d[f"add_{k}_mmm"] = z, g, ctr.mmm
    np.savez_compressed(os.path.join(HERE, "ns.npz"), **d)


def richardson_family():
    rng = np.random.default_rng(103)
    a, eps = contractive(5, 0.99, rng)
    sp = si.split_scalar(a, eps)
    theta_star = rng.standard_normal(5)
    b = a @ theta_star
    bm = rng.standard_normal((5, 3))
    d = {"a": sp.matrix, "precond": sp.precond, "residual": sp.residual, "b": b, "bm": bm}
    for tag, (p, w, n, q, rhs) in {"d22": (0, 1, 2, 2, b), "d23": (0, 1, 2, 3, b),
                                   "d33": (1, 1, 3, 3, b), "m22": (0, 1, 2, 2, bm)}.items():
        st = si.initial_richardson(sp, rhs, p, w, order=n, q=q)
        d[f"{tag}_theta0"], d[f"{tag}_mmm0"], d[f"{tag}_mvm0"] = st.theta, st.ctr.mmm, st.ctr.mvm
        for k in range(3):
            st = si.richardson_step(st, sp.matrix, rhs)
            d[f"{tag}_{k}_theta"], d[f"{tag}_{k}_g"] = st.theta, st.inner.estimate
            d[f"{tag}_{k}_mmm"], d[f"{tag}_{k}_mvm"] = st.ctr.mmm, st.ctr.mvm
    for tag, (p, w, n, rhs) in {"r2": (1, 2, 2, b), "r3": (1, 2, 3, b), "rm2": (0, 1, 2, bm),
                                "r4": (0, 1, 4, b)}.items():
        st = si.initial_richardson(sp, rhs, p, w, order=n, q=n)
        d[f"{tag}_theta0"] = st.theta
        for k in range(4):
            st = si.richardson_recursive_step(st, sp.matrix, rhs)
            d[f"{tag}_{k}_theta"], d[f"{tag}_{k}_omega"] = st.theta, st.omega
            d[f"{tag}_{k}_g"], d[f"{tag}_{k}_l"] = st.inner.estimate, st.inner.accel_estimate
            d[f"{tag}_{k}_mmm"], d[f"{tag}_{k}_mvm"] = st.ctr.mmm, st.ctr.mvm
    np.savez_compressed(os.path.join(HERE, "richardson.npz"), **d)


def plain(theta, p, a, b, ctr):
    """SURVEY a12 with the reference's own products (richardson.py:88-89 ordering)."""
    resid = si.mat_vec(a, theta, ctr) - b
    return theta - si.mat_vec(p, resid, ctr)


def keep(k, iters):
    return k in (1, 2, 3, 5, 10) or k == iters


def config_runs():
    # C1: n=64, NS order 3 + plain Richardson, 30 iterations (full size)
    a, b = configs.c1_dense_small()
    sp = si.split_scalar(a, eps=si.inf_norm(a) / 2.0)
    st = si.initial_series(sp, 0, 1, order=3)
    theta = np.zeros_like(b)
    d = {"a": a, "b": b, "iters": 30}
    for k in range(1, 31):
        theta = plain(theta, st.estimate, sp.matrix, b, st.ctr)
        st = si.ns_step(st, sp.matrix)
        d[f"theta_{k}"], d[f"p_{k}"] = theta, st.estimate
    d["mmm"], d["mvm"] = st.ctr.mmm, st.ctr.mvm
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **d)

    # C2: 4 of the 16384 systems (same recipe), composite (2,3), n=2, 50 iterations
    a2, b2 = configs.c2_batched(batch=4)
    d = {"a": a2, "b": b2, "iters": 50}
    for i in range(a2.shape[0]):
        sp = si.split_scalar(a2[i], eps=si.inf_norm(a2[i]) / 2.0)
        st = si.initial_series(sp, 0, 1, order=2)
        theta = np.zeros(a2.shape[1])
        for k in range(1, 51):
            theta = plain(theta, st.estimate, sp.matrix, b2[i], st.ctr)
            st = si.composite_step(st, sp.matrix, sp, si.CompositeSpec((2, 3)), order_n=2)
            d[f"s{i}_theta_{k}"] = theta
            if keep(k, 50):
                d[f"s{i}_p_{k}"], d[f"s{i}_f_{k}"] = st.estimate, st.residual
        d[f"s{i}_mmm"], d[f"s{i}_mvm"] = st.ctr.mmm, st.ctr.mvm
    np.savez_compressed(os.path.join(HERE, "c2.npz"), **d)

    # C3 (reduced n=128, m=256): order-8 factorised NS (h8) + plain Richardson, 25 iterations
    a, b = configs.c3_gram(n=128)
    sp = si.split_scalar(a, eps=si.inf_norm(a) / 2.0)
    st = si.initial_series(sp, 0, 1, order=8)
    theta = np.zeros_like(b)
    d = {"a": a, "b": b, "iters": 25}
    for k in range(1, 26):
        theta = plain(theta, st.estimate, sp.matrix, b, st.ctr)
        st = si.ns_step(st, sp.matrix, plan=si.table_plans()[8][0])
        d[f"theta_{k}"] = theta
        if keep(k, 25):
            d[f"p_{k}"] = st.estimate
    d["mmm"], d["mvm"] = st.ctr.mmm, st.ctr.mvm
    np.savez_compressed(os.path.join(HERE, "c3.npz"), **d)

    # C4 (reduced n=96, 8 RHS): composite (2,3,4,5), n=2 + plain Richardson, 40 iterations
    a, b = configs.c4_householder(n=96, rhs=8)
    sp = si.split_scalar(a, eps=si.inf_norm(a) / 2.0)
    st = si.initial_series(sp, 0, 1, order=2)
    theta = np.zeros_like(b)
    d = {"a": a, "b": b, "iters": 40}
    for k in range(1, 41):
        theta = plain(theta, st.estimate, sp.matrix, b, st.ctr)
        st = si.composite_step(st, sp.matrix, sp, si.CompositeSpec((2, 3, 4, 5)), order_n=2)
        d[f"theta_{k}"] = theta
        if keep(k, 40):
            d[f"p_{k}"] = st.estimate
    d["mmm"], d["mvm"] = st.ctr.mmm, st.ctr.mvm
    np.savez_compressed(os.path.join(HERE, "c4.npz"), **d)

    # C5 (reduced n=96, m=120, 8 RHS): recursive Richardson/NS order 16, 20 iterations
    n5, m5 = 96, 120
    rng = np.random.default_rng(0)
    g = rng.standard_normal((m5, n5))
    b = rng.standard_normal((n5, 8))
    a = g.T @ g / m5 + 1e-3 * np.eye(n5)
    a = (a + a.T) / 2.0
    sp = si.split_scalar(a, eps=si.inf_norm(a) / 2.0)
    st = si.initial_richardson(sp, b, 0, 1, order=16, q=16)
    d = {"a": a, "b": b, "iters": 20, "theta_0": st.theta}
    for k in range(1, 21):
        st = si.richardson_recursive_step(st, sp.matrix, b)
        d[f"theta_{k}"] = st.theta
        if keep(k, 20):
            d[f"p_{k}"], d[f"omega_{k}"] = st.inner.estimate, st.omega
        d[f"mmm_{k}"] = st.ctr.mmm
    d["mmm"], d["mvm"] = st.ctr.mmm, st.ctr.mvm
    np.savez_compressed(os.path.join(HERE, "c5.npz"), **d)


def harness_runs():
    """run_comparison (harness.py:343-387) + records_to_csv (hx:395-404) on a small
    SPD system, every method kind, with a deterministic injected timer."""
    rng = np.random.default_rng(1234)
    n = 24
    a = spd(n, rng, shift=0.8)
    theta_star = rng.standard_normal(n)
    b = a @ theta_star
    methods = [si.MethodSpec("ns", order=2, h=1), si.MethodSpec("ns", order=3, h=4),
               si.MethodSpec("double", order=2, h=2),
               si.MethodSpec("composite", order=2, h=1, rates=(2, 3)),
               si.MethodSpec("sri", order=2, h=3), si.MethodSpec("ns-estimator", order=2, h=1),
               si.MethodSpec("richardson", order=2, h=1),
               si.MethodSpec("richardson-recursive", order=3, h=2)]
    clock = [0]

    def timer():
        clock[0] += 1000
        return clock[0]

    recs = si.run_comparison(a, b, theta_star, methods, 4, timer=timer)
    out = {"a": a.tolist(), "b": b.tolist(), "theta_star": theta_star.tolist(), "steps": 4,
           "methods": [[m.kind, m.order, m.h, m.q, list(m.rates), m.label] for m in methods],
           "csv": si.records_to_csv(recs),
           "diverged": [bool(r.diverged) for r in recs]}
    # the acceptance criterion-8 run (tests/test_acceptance.py:244-271) on the
    # reference's default harmonic fixture: inputs and the reference's records
    ha, hb, hts = si.gen_harmonic_matrix(si.HarmonicRegressorSpec.default())
    hm = [si.MethodSpec(kind="richardson", order=3, q=3, h=16),
          si.MethodSpec(kind="ns-estimator", order=8, h=16)]
    clock[0] = 0
    hrecs = si.run_comparison(ha, hb, hts, hm, steps=5, eps=0.01 * si.inf_norm(ha), timer=timer)
    out["harmonic"] = {"a": np.asarray(ha).tolist(), "b": np.asarray(hb).tolist(),
                       "theta_star": np.asarray(hts).tolist(),
                       "eps": 0.01 * si.inf_norm(ha), "steps": 5,
                       "methods": [[m.kind, m.order, m.h, m.q, list(m.rates), m.label]
                                   for m in hm],
                       "csv": si.records_to_csv(hrecs)}
    with open(os.path.join(HERE, "harness.json"), "w") as fh:
        json.dump(out, fh)


def setup_family():
    """Setup path: symmetry check + symmetrize (sp:67-73), PD
    verdicts with the pivot floor (sp:76-98), spectral radius (mc:183-239)."""
    from seriesinv.splitting import _check_symmetric

    rng = np.random.default_rng(808)
    d = {}
    # symmetry: relative asymmetry 1e-13 (accepted) / 1e-8 (rejected)
    for i, (dim, rel) in enumerate([(5, 1e-13), (40, 1e-13), (40, 1e-8), (130, 0.0), (130, 1e-7)]):
        a = spd(dim, rng)
        a = a + rel * np.linalg.norm(a) / dim * rng.standard_normal((dim, dim))
        d[f"sym{i}_a"] = a
        try:
            d[f"sym{i}_out"] = _check_symmetric(a)
            d[f"sym{i}_ok"] = np.array(1)
        except ValueError:
            d[f"sym{i}_ok"] = np.array(0)
    # positive definiteness
    cases = [np.eye(3), np.array([[1.0, 2.0], [2.0, 1.0]]), np.zeros((2, 2)),
             np.array([[1.0, 1.0], [1.0, 1.0 + 1e-16]])]
    for dim in (7, 64, 200, 300):
        a = spd(dim, rng)
        cases.append(a)                                    # SPD
        ev_min = float(np.linalg.eigvalsh(a).min())
        cases.append(a - (ev_min + 1e-3) * np.eye(dim))    # indefinite by a clear margin
        cases.append(a - (ev_min - 1e-6) * np.eye(dim))    # SPD, lambda_min = 1e-6
    big = spd(150, rng)
    blk = np.zeros((152, 152))
    blk[:75, :75] = big[:75, :75]
    blk[75:77, 75:77] = [[1.0, 1.0], [1.0, 1.0 + 1e-16]]   # exactly singular pivot mid-matrix
    blk[77:, 77:] = big[75:, 75:]
    cases.append(blk)
    for i, a in enumerate(cases):
        d[f"pd{i}_a"] = a
        d[f"pd{i}_default"] = np.array(int(si.is_positive_definite(a)))
        d[f"pd{i}_zero_tol"] = np.array(int(si.is_positive_definite(a, pivot_tol=0.0)))
    d["pd_count"] = np.array(len(cases))
    # spectral radius
    rads = [np.diag([0.9, 0.1]), np.eye(4), np.zeros((3, 3))]
    for dim in (6, 50, 200):
        q, _ = np.linalg.qr(rng.standard_normal((dim, dim)))
        ev = rng.uniform(-0.5, 0.5, dim)
        ev[0] = 0.95
        rads.append((q * ev) @ q.T)
    for i, m in enumerate(rads):
        d[f"rho{i}_a"] = m
        d[f"rho{i}"] = np.array(si.spectral_radius(m))
    d["rho_count"] = np.array(len(rads))
    np.savez_compressed(os.path.join(HERE, "setup.npz"), **d)


if __name__ == "__main__":
    if sys.argv[1:] == ["setup"]:  # regenerate only setup.npz
        setup_family()
        sys.exit(0)
    setup_family()
    harness_runs()
    plans_json()
    toolkit()
    ns_family()
    richardson_family()
    config_runs()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
