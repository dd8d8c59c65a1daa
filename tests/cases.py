"""Golden-case drivers shared by the oracle tests (CPU) and the parity tests (GPU).

Each ``case_*`` function replays one block of tests/golden/make_golden.py
through a backend ``B`` (the numpy oracle, or the CUDA library) and returns
{golden key: value}; the tests compare those against the stored fixtures.
"""

from __future__ import annotations

import numpy as np

from conftest import golden

KEEP = (1, 2, 3, 5, 10)


class OracleBackend:
    """The CPU oracle (oracle/seriesinv_oracle.py) -- checker only."""

    name = "oracle"

    def __init__(self):
        from oracle import seriesinv_oracle as o

        self.o = o

    def counter(self):
        return self.o.Counter()

    def np(self, x):
        return np.asarray(x)

    def dev(self, x):
        return np.asarray(x, dtype=np.float64)

    # plans
    def plan_order(self, h):
        return self.o.plan_order(h)

    def table_plan(self, order, idx):
        return self.o.TABLE_ROOTS[order][idx][1]

    def table_items(self):
        for order, rows in self.o.TABLE_ROOTS.items():
            for label, node in rows:
                yield order, label, node

    def order45(self):
        return self.o.order45()

    # primitives
    def mat_mul(self, a, b, c):
        return self.o.mm(a, b, c)

    def mat_pow_counted(self, y, e, c):
        return self.o.mat_pow_counted(y, e, c)

    def horner_eval(self, y, x, h, c, a=None, form_y=False):
        return self.o.horner_eval(y, x, h, c, a=a, form_y=form_y)

    def factored_eval(self, y, x, a, p, w, c, form_y):
        return self.o.factored_eval(y, x, a, p, w, c, form_y=form_y)

    def nested_eval(self, y, x, a, plan, c, form_y=True):
        return self.o.nested_eval(y, x, a, plan, c, form_y=form_y)

    def geometric_apply(self, y, x, order, a, c):
        return self.o.geometric_apply(y, x, order, a, c)

    # splittings and steps
    def split_scalar(self, a, eps):
        return self.o.split_scalar(a, eps)

    def split_diagonal(self, a):
        return self.o.split_diagonal(a)

    def initial_series(self, sp, p, w, order):
        return self.o.initial_series(sp, p, w, order)

    def ns_step(self, st, a, plan=None):
        return self.o.ns_step(st, a, plan)

    def composite_step(self, st, a, sp, rates, n):
        return self.o.composite_step(st, a, sp, rates, n)

    def initial_double(self, sp, p, w, order):
        return self.o.initial_double(sp, p, w, order)

    def double_ns_step(self, st, a):
        return self.o.double_ns_step(st, a)

    def additive(self, z, g, a, p, c):
        return self.o.additive_correction_step(z, g, a, p, c)

    def initial_richardson(self, sp, b, p, w, order, q):
        return self.o.initial_richardson(sp, b, p, w, order, q)

    def richardson_step(self, st, a, b):
        return self.o.richardson_step(st, a, b)

    def richardson_recursive_step(self, st, a, b):
        return self.o.richardson_recursive_step(st, a, b)

    def plain(self, theta, p, a, b, c):
        return self.o.plain_richardson(theta, p, a, b, c)

    def inf_norm(self, a):
        return self.o.inf_norm(a)


def case_toolkit(B):
    g = golden("toolkit.npz")
    a, x, y = B.dev(g["a"]), B.dev(g["x"]), B.dev(g["y"])
    out = {}
    for h in (1, 2, 3, 8):
        c = B.counter()
        out[f"horner_{h}"] = B.horner_eval(y, x, h, c)
        out[f"horner_{h}_mmm"] = c.mmm
        c = B.counter()
        out[f"hornerf_{h}"] = B.horner_eval(y, x, h, c, a=a, form_y=True)
        out[f"hornerf_{h}_mmm"] = c.mmm
    for p, w in ((0, 1), (1, 1), (1, 2), (2, 3), (3, 4), (0, 3)):
        for fy in (True, False):
            c = B.counter()
            out[f"factored_{p}_{w}_{int(fy)}"] = B.factored_eval(y, x, a, p, w, c, fy)
            out[f"factored_{p}_{w}_{int(fy)}_mmm"] = c.mmm
    for h in range(2, 65):
        c = B.counter()
        out[f"plan_{h}"] = B.nested_eval(y, x, a, B.plan_order(h), c)
        out[f"plan_{h}_mmm"] = c.mmm
    for order, label, plan in B.table_items():
        c = B.counter()
        out[f"table_{label}"] = B.nested_eval(y, x, a, plan, c, form_y=False)
        out[f"table_{label}_mmm"] = c.mmm
    c = B.counter()
    out["order45"] = B.nested_eval(y, x, a, B.order45(), c)
    out["order45_mmm"] = c.mmm
    for order in (1, 2, 3, 19, 20, 64, 65, 130, 200):
        c = B.counter()
        out[f"geom_{order}"] = B.geometric_apply(y, x, order, a, c)
        out[f"geom_{order}_mmm"] = c.mmm
    for e in (0, 1, 5, 6, 13):
        c = B.counter()
        out[f"pow_{e}"] = B.mat_pow_counted(y, e, c)
        out[f"pow_{e}_mmm"] = c.mmm
    out["mm_ab"] = B.mat_mul(B.dev(g["mm_a"]), B.dev(g["mm_b"]), B.counter())
    return out


def case_ns(B):
    g = golden("ns.npz")
    a = B.dev(g["a"])
    sp = B.split_diagonal(a)
    out = {}
    for p, w, n in ((0, 1, 2), (1, 1, 3), (1, 2, 2), (2, 3, 4)):
        st = B.initial_series(sp, p, w, n)
        key = f"init_{p}_{w}"
        out[key + "_g"], out[key + "_f"], out[key + "_mmm"] = st.estimate, st.residual, st.ctr.mmm
        for k in range(3):
            st = B.ns_step(st, sp.matrix)
            out[f"ns_{p}_{w}_{n}_{k}_g"] = st.estimate
            out[f"ns_{p}_{w}_{n}_{k}_f"] = st.residual
            out[f"ns_{p}_{w}_{n}_{k}_mmm"] = st.ctr.mmm
    st = B.initial_series(sp, 0, 1, 8)
    for k in range(2):
        st = B.ns_step(st, sp.matrix, B.table_plan(8, 0))
        out[f"nsh8_{k}_g"], out[f"nsh8_{k}_f"], out[f"nsh8_{k}_mmm"] = st.estimate, st.residual, st.ctr.mmm
    for tag, rates, n in (("c23", (2, 3), 2), ("c2345", (2, 3, 4, 5), 2), ("c1", (1,), 1),
                          ("c100", (100,), 2), ("c22", (2, 2), 3)):
        st = B.initial_series(sp, 0, 1, n)
        for k in range(2):
            st = B.composite_step(st, sp.matrix, sp, rates, n)
            out[f"comp_{tag}_{k}_g"], out[f"comp_{tag}_{k}_f"] = st.estimate, st.residual
            out[f"comp_{tag}_{k}_mmm"] = st.ctr.mmm
    dst = B.initial_double(sp, 1, 2, 3)
    out["dbl_init_g"], out["dbl_init_f"] = dst.estimate, dst.residual
    out["dbl_init_l"], out["dbl_init_r"], out["dbl_init_mmm"] = (
        dst.accel_estimate, dst.accel_residual, dst.ctr.mmm)
    for k in range(3):
        dst = B.double_ns_step(dst, sp.matrix)
        for f, v in (("g", dst.estimate), ("f", dst.residual), ("l", dst.accel_estimate),
                     ("r", dst.accel_residual)):
            out[f"dbl_{k}_{f}"] = v
        out[f"dbl_{k}_mmm"] = dst.ctr.mmm
    z = gg = sp.precond
    c = B.counter()
    for k in range(2):
        z, gg = B.additive(z, gg, sp.matrix, 3, c)
        out[f"add_{k}_z"], out[f"add_{k}_g"], out[f"add_{k}_mmm"] = z, gg, c.mmm
    return out


def case_richardson(B):
    g = golden("richardson.npz")
    a = B.dev(g["a"])
    # alpha = 1 in the fixture: eps = 1 - ||A||_inf / 2
    sp = B.split_scalar(a, 1.0 - B.inf_norm(a) / 2.0)
    b, bm = B.dev(g["b"]), B.dev(g["bm"])
    out = {}
    for tag, (p, w, n, q, rhs) in {"d22": (0, 1, 2, 2, b), "d23": (0, 1, 2, 3, b),
                                   "d33": (1, 1, 3, 3, b), "m22": (0, 1, 2, 2, bm)}.items():
        st = B.initial_richardson(sp, rhs, p, w, n, q)
        out[f"{tag}_theta0"], out[f"{tag}_mmm0"], out[f"{tag}_mvm0"] = st.theta, st.ctr.mmm, st.ctr.mvm
        for k in range(3):
            st = B.richardson_step(st, sp.matrix, rhs)
            out[f"{tag}_{k}_theta"], out[f"{tag}_{k}_g"] = st.theta, st.inner.estimate
            out[f"{tag}_{k}_mmm"], out[f"{tag}_{k}_mvm"] = st.ctr.mmm, st.ctr.mvm
    for tag, (p, w, n, rhs) in {"r2": (1, 2, 2, b), "r3": (1, 2, 3, b), "rm2": (0, 1, 2, bm),
                                "r4": (0, 1, 4, b)}.items():
        st = B.initial_richardson(sp, rhs, p, w, n, n)
        out[f"{tag}_theta0"] = st.theta
        for k in range(4):
            st = B.richardson_recursive_step(st, sp.matrix, rhs)
            out[f"{tag}_{k}_theta"], out[f"{tag}_{k}_omega"] = st.theta, st.omega
            out[f"{tag}_{k}_g"], out[f"{tag}_{k}_l"] = st.inner.estimate, st.inner.accel_estimate
            out[f"{tag}_{k}_mmm"], out[f"{tag}_{k}_mvm"] = st.ctr.mmm, st.ctr.mvm
    return out


def _dense_run(B, fixture, make_state, step, every_theta=True):
    g = golden(fixture)
    a, b = B.dev(g["a"]), B.dev(g["b"])
    sp = B.split_scalar(a, B.inf_norm(a) / 2.0)
    st = make_state(sp)
    theta = B.dev(np.zeros(g["b"].shape))
    iters = int(g["iters"])
    out = {}
    for k in range(1, iters + 1):
        theta = B.plain(theta, st.estimate, sp.matrix, b, st.ctr)
        st = step(st, sp)
        out[f"theta_{k}"] = theta
        if k in KEEP or k == iters:
            out[f"p_{k}"] = st.estimate
    out["mmm"], out["mvm"] = st.ctr.mmm, st.ctr.mvm
    return out


def case_c1(B):
    return _dense_run(B, "c1.npz", lambda sp: B.initial_series(sp, 0, 1, 3),
                      lambda st, sp: B.ns_step(st, sp.matrix))


def case_c3(B):
    return _dense_run(B, "c3.npz", lambda sp: B.initial_series(sp, 0, 1, 8),
                      lambda st, sp: B.ns_step(st, sp.matrix, B.table_plan(8, 0)))


def case_c4(B):
    return _dense_run(B, "c4.npz", lambda sp: B.initial_series(sp, 0, 1, 2),
                      lambda st, sp: B.composite_step(st, sp.matrix, sp, (2, 3, 4, 5), 2))


def case_c5(B):
    g = golden("c5.npz")
    a, b = B.dev(g["a"]), B.dev(g["b"])
    sp = B.split_scalar(a, B.inf_norm(a) / 2.0)
    st = B.initial_richardson(sp, b, 0, 1, 16, 16)
    out = {"theta_0": st.theta}
    for k in range(1, 21):
        st = B.richardson_recursive_step(st, sp.matrix, b)
        out[f"theta_{k}"] = st.theta
        if k in KEEP or k == 20:
            out[f"p_{k}"], out[f"omega_{k}"] = st.inner.estimate, st.omega
        out[f"mmm_{k}"] = st.ctr.mmm
    out["mmm"], out["mvm"] = st.ctr.mmm, st.ctr.mvm
    return out


def case_c2_oracle(B):
    """Per-system oracle replay of the batched fixture (4 systems)."""
    g = golden("c2.npz")
    out = {}
    for i in range(g["a"].shape[0]):
        a, b = B.dev(g["a"][i]), B.dev(g["b"][i])
        sp = B.split_scalar(a, B.inf_norm(a) / 2.0)
        st = B.initial_series(sp, 0, 1, 2)
        theta = B.dev(np.zeros(a.shape[0]))
        for k in range(1, 51):
            theta = B.plain(theta, st.estimate, sp.matrix, b, st.ctr)
            st = B.composite_step(st, sp.matrix, sp, (2, 3), 2)
            out[f"s{i}_theta_{k}"] = theta
            if k in KEEP or k == 50:
                out[f"s{i}_p_{k}"], out[f"s{i}_f_{k}"] = st.estimate, st.residual
        out[f"s{i}_mmm"], out[f"s{i}_mvm"] = st.ctr.mmm, st.ctr.mvm
    return out


def compare(out: dict, fixture: str, B, rtol: float, ftol: float | None = None):
    """Check every produced key against the fixture.  Integers (counters) are
    exact; estimates/thetas use relative Frobenius error <= rtol; residual-like
    keys (``_f``/``_r``, which converge to 0) use ||delta||_F <= ftol * sqrt(n)."""
    g = golden(fixture)
    worst = 0.0
    for key, val in out.items():
        assert key in g.files, f"{key} missing from {fixture}"
        ref = g[key]
        if ref.dtype.kind in "iu":
            assert int(val) == int(ref), f"{fixture}:{key}: {int(val)} != {int(ref)}"
            continue
        v = B.np(val)
        assert v.shape == ref.shape, f"{fixture}:{key}: shape {v.shape} != {ref.shape}"
        if ftol is not None and (key.endswith("_f") or key.endswith("_r") or "_f_" in key):
            err = float(np.linalg.norm(v - ref)) / np.sqrt(max(ref.shape[0], 1))
            assert err <= ftol, f"{fixture}:{key}: abs err {err:.3e} > {ftol:.1e}"
            continue
        den = float(np.linalg.norm(ref))
        err = float(np.linalg.norm(v - ref)) / (den if den > 0 else 1.0)
        worst = max(worst, err)
        assert err <= rtol, f"{fixture}:{key}: rel err {err:.3e} > {rtol:.1e}"
    return worst
