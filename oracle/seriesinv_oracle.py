"""CPU oracle for the seriesinv hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it.  The CUDA path in ``paper_2008_11480_b200``
never routes through here.

It is a numpy restatement of the reference package ``seriesinv``
(``/root/reference/pkg/src/seriesinv``), whose arithmetic is numpy ``@``
(OpenBLAS dgemm/dgemv) plus element-wise temporaries.  Every function cites the
reference ``file:line`` it follows; the GEMM DAG (order of products, which
products are counted, how the element-wise terms are rounded) is kept
identical so that the multiplication counters match and results agree to the
FP64 noise floor.

Pinning: ``tests/golden/`` holds vectors produced by importing the real
reference in the build container (``tests/golden/make_golden.py``);
``tests/test_oracle_golden.py`` checks this restatement against them.

Abbreviations: mc = matrix_core.py, st = series_toolkit.py,
ns = newton_schulz.py, ri = richardson.py, sp = splitting.py.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

# ---------------------------------------------------------------------------
# L1: counted products (mc:71-114)
# ---------------------------------------------------------------------------


@dataclass
class Counter:
    """mmm / mvm tallies (mc:71-98)."""

    mmm: int = 0
    mvm: int = 0

    def merge(self, other: "Counter") -> None:
        self.mmm += other.mmm
        self.mvm += other.mvm


def mm(a, b, ctr: Counter):
    """mc:101-106 -- ``a @ b`` with one mmm tick."""
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"dimension mismatch: {a.shape} @ {b.shape}")
    ctr.mmm += 1
    return a @ b


def mv(a, v, ctr: Counter):
    """mc:109-114 -- ``a @ v`` (v may be n x r) with one mvm tick."""
    if a.shape[1] != v.shape[0]:
        raise ValueError(f"dimension mismatch: {a.shape} @ {v.shape}")
    ctr.mvm += 1
    return a @ v


def eye(n):
    return np.eye(n, dtype=np.float64)


def fro(a) -> float:
    """mc:154-168 -- sqrt(sum(a*a))."""
    return float(np.sqrt(np.sum(a * a)))


def inf_norm(a) -> float:
    """mc:154-172 -- max row sum of |a|."""
    return float(np.max(np.sum(np.abs(a), axis=1)))


def mat_pow(a, e: int):
    """mc:117-134 -- uncounted binary exponentiation (exponent-law oracle)."""
    out = eye(a.shape[0])
    base = np.array(a)
    while e > 0:
        if e & 1:
            out = out @ base
        e >>= 1
        if e:
            base = base @ base
    return out


def mat_pow_counted(a, e: int, ctr: Counter):
    """mc:137-151 -- counted binary exponentiation."""
    if e == 0:
        return eye(a.shape[0])
    base, out = np.array(a), None
    while e > 0:
        if e & 1:
            out = base if out is None else mm(out, base, ctr)
        e >>= 1
        if e:
            base = mm(base, base, ctr)
    return out


# ---------------------------------------------------------------------------
# L2: splittings (sp:42-146)
# ---------------------------------------------------------------------------


@dataclass
class Split:
    """sp:42-64 -- S^-1 (precond), B = I - S^-1 A (residual), A (matrix)."""

    precond: np.ndarray
    residual: np.ndarray
    matrix: np.ndarray
    kind: str


def _symmetrize(a):
    """sp:67-73 -- reject asymmetric input, return (a + a.T)/2."""
    a = np.array(a, dtype=np.float64)
    if fro(a - a.T) > 1e-10 * max(fro(a), 1e-300):
        raise ValueError("matrix must be symmetric")
    return (a + a.T) / 2.0


def check_symmetric(a):
    """sp:67-73 -- (||A - A^T||_F, ||A||_F, (A + A^T)/2); the caller rejects
    asym > 1e-10 max(fro, 1e-300) (sp:70-71)."""
    a = np.array(a, dtype=np.float64)
    return fro(a - a.T), fro(a), (a + a.T) / 2.0


def is_positive_definite(a, pivot_tol=None) -> bool:
    """sp:76-98 -- left-looking Cholesky of (a + a^T)/2; a pivot d <= pivot_tol
    (default 1e-12 ||a||_inf) means not PD.  Python loop over columns: for
    n in the hundreds (use is_positive_definite_blocked above that)."""
    a = np.array(a, dtype=np.float64)
    a = (a + a.T) / 2.0
    n = a.shape[0]
    if pivot_tol is None:
        pivot_tol = 1e-12 * inf_norm(a)
    lower = np.zeros_like(a)
    for j in range(n):
        d = a[j, j] - np.dot(lower[j, :j], lower[j, :j])
        if d <= pivot_tol:
            return False
        lower[j, j] = np.sqrt(d)
        if j + 1 < n:
            lower[j + 1:, j] = (a[j + 1:, j] - lower[j + 1:, :j] @ lower[j, :j]) / lower[j, j]
    return True


def is_positive_definite_blocked(a, pivot_tol=None, nb: int = 256) -> bool:
    """The same test as :func:`is_positive_definite` (sp:76-98) for large n:
    right-looking blocked Cholesky in numpy/LAPACK (the diagonal blocks by the
    column loop, panels by triangular solves, trailing updates by BLAS), the
    same pivot floor on every pivot.  Pivots equal the loop's up to rounding, so
    the verdict agrees on every input whose smallest pivot is not within
    rounding of the floor."""
    a = np.array(a, dtype=np.float64)
    a = (a + a.T) / 2.0
    n = a.shape[0]
    if pivot_tol is None:
        pivot_tol = 1e-12 * inf_norm(a)
    for k in range(0, n, nb):
        e = min(n, k + nb)
        blk = a[k:e, k:e]
        lk = np.zeros_like(blk)
        for j in range(e - k):
            d = blk[j, j] - np.dot(lk[j, :j], lk[j, :j])
            if d <= pivot_tol:
                return False
            lk[j, j] = np.sqrt(d)
            if j + 1 < e - k:
                lk[j + 1:, j] = (blk[j + 1:, j] - lk[j + 1:, :j] @ lk[j, :j]) / lk[j, j]
        if e < n:
            import scipy.linalg as sla

            w = sla.solve_triangular(lk, a[e:, k:e].T, lower=True).T  # A21 L11^-T
            a[e:, e:] -= w @ w.T
    return True


def spectral_radius(a, tol=1e-12, max_iter=10000, seed=0) -> float:
    """mc:183-239 -- norm-ratio power iteration, restarts on est == 0; raises
    RuntimeError with the best estimate when it does not settle."""
    dim = a.shape[0]
    rng = np.random.default_rng(seed)
    best, restarts = 0.0, 0
    x = rng.standard_normal(dim)
    x /= np.linalg.norm(x)
    prev, streak = None, 0
    for _ in range(max_iter):
        y = a @ x
        est = float(np.linalg.norm(y))
        if est == 0.0:
            if not np.any(a):
                return 0.0
            restarts += 1
            if restarts > 3:
                return 0.0
            x = rng.standard_normal(dim)
            x /= np.linalg.norm(x)
            prev, streak = None, 0
            continue
        best = est
        if prev is not None and abs(est - prev) <= tol * est:
            streak += 1
            if streak >= 3:
                return est
        else:
            streak = 0
        prev = est
        x = y / est
    raise RuntimeError(f"power iteration did not converge (best estimate {best:.6e})")


def split_scalar(a, eps=None) -> Split:
    """sp:124-146 -- S^-1 = I/alpha, alpha = ||A||_inf/2 + eps (PD check skipped:
    the oracle is only fed SPD fixtures)."""
    a = _symmetrize(a)
    if eps is None:
        eps = 1e-3 * inf_norm(a)
    alpha = inf_norm(a) / 2.0 + eps
    n = a.shape[0]
    return Split(eye(n) / alpha, eye(n) - a / alpha, a, "scalar")


def split_diagonal(a) -> Split:
    """sp:101-121 -- S = diag(A)."""
    a = _symmetrize(a)
    d = np.diag(a)
    n = a.shape[0]
    return Split(np.diag(1.0 / d), eye(n) - a / d[:, None], a, "diagonal")


# ---------------------------------------------------------------------------
# L3: plans and evaluators (st:71-747)
# Plan nodes are tuples: ("horner", h) | ("split", p, w, inner, outer)
# | ("wrap", inner) | ("table", label, order, program).  Program instructions:
# ("mul", dst, lhs, rhs) | ("res", dst, src) | ("lin", dst, const, ((coef, reg), ...)).
# ---------------------------------------------------------------------------


def node_order(node) -> int:
    """st:165-192."""
    kind = node[0]
    if kind == "horner":
        return node[1]
    if kind == "split":
        return node[2] * (node[1] + 1)
    if kind == "wrap":
        return node_order(node[1]) + 1
    return node[2]


def node_poly_cost(node) -> int:
    """st:195-207."""
    kind = node[0]
    if kind == "horner":
        return node[1] - 1
    if kind == "split":
        _, p, w, inner, outer = node
        c = 0 if p == 0 else node_poly_cost(inner)
        if w >= 2:
            c += (0 if p == 0 else 1) + node_poly_cost(outer)
        return c
    if kind == "wrap":
        return node_poly_cost(node[1]) + 1
    return sum(1 for ins in node[3] if ins[0] in ("mul", "res"))


def node_depth(node) -> int:
    """st:210-221."""
    kind = node[0]
    if kind == "horner":
        return 0
    if kind == "split":
        outer = node_depth(node[4]) if node[4] is not None else 0
        return 1 + max(node_depth(node[3]), outer)
    if kind == "wrap":
        return node_depth(node[1])
    return 1


def node_str(node) -> str:
    """st:240-255 canonical text form."""
    kind = node[0]
    if kind == "horner":
        return f"horner(h={node[1]})"
    if kind == "split":
        _, p, w, inner, outer = node
        parts = [f"p={p},w={w}"]
        if p >= 1 and inner[0] != "horner":
            parts.append(f"inner={node_str(inner)}")
        if w >= 2 and outer is not None and outer[0] != "horner":
            parts.append(f"outer={node_str(outer)}")
        return "split(" + ", ".join(parts) + ")"
    if kind == "wrap":
        return f"wrap({node_str(node[1])})"
    return f"table({node[1]})"


def _mul(d, l, r):
    return ("mul", d, l, r)


def _res(d, s):
    return ("res", d, s)


def _lin(d, c, *regs):
    return ("lin", d, c, tuple((1.0, r) for r in regs))


# The folded table forms (st:465-618), as straight-line programs over Y, X.
TABLE_FORMS = {
    "h5b": ("table", "h5b", 5, (
        _mul("y2", "Y", "Y"), _lin("s", 0.0, "Y", "y2"), _mul("t", "y2", "s"),
        _lin("m", 1.0, "Y", "y2", "t"), _mul("z", "m", "X"))),
    "h7": ("table", "h7", 7, (
        _mul("y2", "Y", "Y"), _mul("y4", "y2", "y2"), _lin("f1", 0.0, "Y", "y4"),
        _lin("f2", 1.0, "Y", "y2"), _mul("w", "f1", "f2"), _mul("t", "w", "X"),
        _lin("z", 0.0, "X", "t"))),
    "h8": ("table", "h8", 8, (
        _mul("c0", "Y", "X"), _lin("c1", 0.0, "X", "c0"), _res("q2", "c1"),
        _mul("c2", "q2", "c1"), _lin("c3", 0.0, "c1", "c2"), _res("q4", "c3"),
        _mul("c4", "q4", "c3"), _lin("z", 0.0, "c3", "c4"))),
    "h9b": ("table", "h9b", 9, (
        _mul("y2", "Y", "Y"), _mul("y4", "y2", "y2"), _lin("f1", 0.0, "Y", "y2"),
        _lin("f2", 1.0, "y2"), _mul("w1", "f2", "f1"), _lin("f3", 1.0, "y4"),
        _mul("w2", "f3", "w1"), _mul("t", "w2", "X"), _lin("z", 0.0, "X", "t"))),
    "h10b": ("table", "h10b", 10, (
        _mul("y2", "Y", "Y"), _lin("f1", 0.0, "Y", "y2"), _lin("f2", 1.0, "y2"),
        _mul("w", "f1", "f2"), _mul("t0", "w", "X"), _lin("u", 0.0, "X", "t0"),
        _res("q5", "u"), _mul("t1", "q5", "u"), _lin("z", 0.0, "u", "t1"))),
    "h11b": ("table", "h11b", 11, (
        _mul("t0", "Y", "X"), _lin("t1", 0.0, "X", "t0"), _res("y2", "t1"),
        _mul("y4", "y2", "y2"), _lin("f1", 0.0, "y2", "y4"), _lin("f2", 1.0, "y4"),
        _mul("w", "f1", "f2"), _mul("t2", "w", "t1"), _lin("t3", 0.0, "t1", "t2"),
        _mul("t4", "Y", "t3"), _lin("z", 0.0, "X", "t4"))),
    "h15b": ("table", "h15b", 15, (
        _mul("c0", "Y", "X"), _lin("c1", 0.0, "X", "c0"), _mul("c2", "Y", "c1"),
        _lin("u", 0.0, "X", "c2"), _res("q3", "u"), _mul("q6", "q3", "q3"),
        _lin("f1", 1.0, "q6"), _lin("f2", 0.0, "q3", "q6"), _mul("w", "f1", "f2"),
        _mul("t", "w", "u"), _lin("z", 0.0, "u", "t"))),
    "h17": ("table", "h17", 17, (
        _mul("y2", "Y", "Y"), _lin("f1", 0.0, "Y", "y2"), _lin("f2", 1.0, "y2"),
        _mul("g", "f1", "f2"), _mul("y4", "y2", "y2"), _mul("y8", "y4", "y4"),
        _mul("y12", "y8", "y4"), _lin("f3", 1.0, "y4", "y8", "y12"),
        _mul("w", "g", "f3"), _mul("t", "w", "X"), _lin("z", 0.0, "X", "t"))),
    "h19": ("table", "h19", 19, (
        _mul("y2", "Y", "Y"), _mul("y4", "y2", "y2"), _lin("f1", 0.0, "Y", "y2"),
        _lin("f2", 1.0, "y2", "y4"), _mul("w1", "f1", "f2"), _mul("y6", "y2", "y4"),
        _mul("y12", "y6", "y6"), _lin("f3", 1.0, "y6", "y12"), _mul("w2", "w1", "f3"),
        _mul("t", "w2", "X"), _lin("z", 0.0, "X", "t"))),
}


def _sp(p, w):
    """st:621-623 -- plain two-level split with Horner leaves."""
    return ("split", p, w, ("horner", p + 1), ("horner", w) if w >= 2 else None)


# st:632-651 -- catalogue rows, order -> ((label, node), ...)
TABLE_ROOTS = {
    2: (("h2", _sp(1, 1)),),
    3: (("h3", ("wrap", _sp(1, 1))),),
    4: (("h4", _sp(1, 2)),),
    5: (("h5a", ("wrap", _sp(1, 2))), ("h5b", TABLE_FORMS["h5b"])),
    6: (("h6", _sp(2, 2)),),
    7: (("h7", TABLE_FORMS["h7"]),),
    8: (("h8", TABLE_FORMS["h8"]),),
    9: (("h9a", _sp(2, 3)), ("h9b", TABLE_FORMS["h9b"])),
    10: (("h10a", ("wrap", _sp(2, 3))), ("h10b", TABLE_FORMS["h10b"])),
    11: (("h11a", ("wrap", TABLE_FORMS["h10b"])), ("h11b", TABLE_FORMS["h11b"])),
    12: (("h12", _sp(3, 3)),),
    13: (("h13", ("wrap", _sp(3, 3))),),
    14: (("h14", _sp(6, 2)),),
    15: (("h15a", _sp(2, 5)), ("h15b", TABLE_FORMS["h15b"])),
    16: (("h16", _sp(3, 4)),),
    17: (("h17", TABLE_FORMS["h17"]),),
    18: (("h18", _sp(5, 3)),),
    19: (("h19", TABLE_FORMS["h19"]),),
}


def order45():
    """st:667-676."""
    return ("split", 8, 5, ("split", 2, 3, ("horner", 3), ("horner", 3)), TABLE_FORMS["h5b"])


def _is_prime(n):
    return n >= 2 and all(n % d for d in range(2, int(n**0.5) + 1))


@lru_cache(maxsize=None)
def _best(h: int, budget: int):
    """st:706-735 -- min (poly cost, rank, p, depth) over Horner, table rows,
    splits over divisor pairs (nested, budget-limited) and prime wraps."""
    cands = [(h - 1, 3, 10**9, 0, ("horner", h))]
    if budget >= 1:
        for _, root in TABLE_ROOTS.get(h, ()):
            cands.append((node_poly_cost(root), 2, 10**9, node_depth(root), root))
        if h == 2:
            cands.append((1, 0, 1, 1, ("split", 1, 1, ("horner", 2), None)))
        for d in range(2, h // 2 + 1):
            if h % d:
                continue
            p, w = d - 1, h // d
            ic, _, _, idp, inner = _best(p + 1, budget - 1)
            oc, _, _, odp, outer = _best(w, budget - 1)
            cands.append((ic + 1 + oc, 0, p, 1 + max(idp, odp), ("split", p, w, inner, outer)))
        if _is_prime(h) and h >= 3:
            ic, _, _, idp, inner = _best(h - 1, budget)
            cands.append((ic + 1, 1, 10**9, idp, ("wrap", inner)))
    return min(cands, key=lambda c: c[:4])


def plan_order(h: int):
    """st:738-747 -- minimal-count plan node of order 2..64."""
    if h < 2 or h > 64:
        raise ValueError("plan_order supports 2 <= h <= 64")
    return _best(h, 3)[4]


def _horner(y, x, h, ctr):
    """st:263-267 -- z <- y z + x, h-1 times."""
    z = x
    for _ in range(h - 1):
        z = mm(y, z, ctr) + x
    return z


def _run_program(prog, y, x, a, ctr):
    """st:359-382 -- straight-line program interpreter."""
    n = x.shape[0]
    env = {"Y": y, "X": x}
    dst = "X"
    for ins in prog:
        if ins[0] == "mul":
            env[ins[1]] = mm(env[ins[2]], env[ins[3]], ctr)
        elif ins[0] == "res":
            env[ins[1]] = eye(n) - mm(env[ins[2]], a, ctr)
        else:
            _, d, const, terms = ins
            acc = const * eye(n) if const else np.zeros_like(x)
            for coef, reg in terms:
                acc = acc + coef * env[reg]
            env[d] = acc
        dst = ins[1]
    return env[dst]


def eval_node(node, y, x, a, ctr):
    """st:385-405."""
    kind = node[0]
    if kind == "horner":
        return _horner(y, x, node[1], ctr)
    if kind == "split":
        _, p, w, inner, outer = node
        u = x if p == 0 else eval_node(inner, y, x, a, ctr)
        if w == 1:
            return u
        q = y if p == 0 else eye(x.shape[0]) - mm(u, a, ctr)
        return eval_node(outer, q, u, a, ctr)
    if kind == "wrap":
        z = eval_node(node[1], y, x, a, ctr)
        return x + mm(y, z, ctr)
    return _run_program(node[3], y, x, a, ctr)


def horner_eval(y, x, h, ctr, a=None, form_y=False):
    """st:279-302."""
    if form_y:
        y = eye(x.shape[0]) - mm(x, a, ctr)
    return _horner(y, x, h, ctr)


def factored_eval(y, x, a, p, w, ctr, form_y=True):
    """st:326-356."""
    if form_y:
        y = eye(x.shape[0]) - mm(x, a, ctr)
    u = x if p == 0 else _horner(y, x, p + 1, ctr)
    if w == 1:
        return u
    q = y if p == 0 else eye(x.shape[0]) - mm(u, a, ctr)
    return _horner(q, u, w, ctr)


def nested_eval(y, x, a, node, ctr, form_y=True):
    """st:408-429."""
    if form_y:
        y = eye(x.shape[0]) - mm(x, a, ctr)
    return eval_node(node, y, x, a, ctr)


def geometric_apply(y, x, order, a, ctr):
    """st:432-457 -- plan_order for order <= 64, doubling beyond."""
    if order == 1:
        return np.array(x)
    if order <= 64:
        return eval_node(plan_order(order), y, x, a, ctr)
    half = order // 2
    t = geometric_apply(y, x, half, a, ctr)
    yh = mat_pow_counted(y, half, ctr)
    z = t + mm(yh, t, ctr)
    if order % 2:
        z = x + mm(y, z, ctr)
    return z


# ---------------------------------------------------------------------------
# L4: Newton-Schulz steps (ns:58-325).  States are plain dicts of arrays.
# ---------------------------------------------------------------------------


@dataclass
class NS:
    """ns:58-72 (estimate G, residual F)."""

    estimate: np.ndarray
    residual: np.ndarray
    step: int
    order: int
    series_order: int
    ctr: Counter


@dataclass
class DoubleNS:
    """ns:75-91."""

    estimate: np.ndarray
    residual: np.ndarray
    accel_estimate: np.ndarray
    accel_residual: np.ndarray
    step: int
    order: int
    series_order: int
    ctr: Counter


def initial_series(sp: Split, p: int, w: int, order: int = 2) -> NS:
    """ns:127-147."""
    h = w * (p + 1)
    ctr = Counter()
    if h == 1:
        g, f = np.array(sp.precond), np.array(sp.residual)
    else:
        g = factored_eval(sp.residual, sp.precond, sp.matrix, p, w, ctr, form_y=False)
        f = eye(g.shape[0]) - mm(g, sp.matrix, ctr)
    return NS(g, f, 0, order, h, ctr)


def ns_step(st: NS, a, plan=None) -> NS:
    """ns:150-174 -- Horner (or a plan node of order n) then F = I - G A."""
    n = st.order
    if plan is None:
        g = _horner(st.residual, st.estimate, n, st.ctr)
    else:
        g = eval_node(plan, st.residual, st.estimate, a, st.ctr)
    f = eye(g.shape[0]) - mm(g, a, st.ctr)
    return NS(g, f, st.step + 1, n, st.series_order, st.ctr)


def composite_step(st: NS, a, sp: Split, rates, order_n: int) -> NS:
    """ns:177-228 -- parts T_i, Gamma_i; left fold; NS part; assembly."""
    ctr = st.ctr
    I = eye(a.shape[0])
    ts, gs = [], []
    for x in rates:
        t = np.array(sp.precond) if x == 1 else geometric_apply(sp.residual, sp.precond, x, sp.matrix, ctr)
        ts.append(t)
        gs.append(I - mm(t, a, ctr))
    t_c, r_c = ts[0], gs[0]
    for i in range(1, len(ts)):
        t_c = t_c + mm(r_c, ts[i], ctr)
        r_c = mm(r_c, gs[i], ctr)
    nsp = _horner(st.residual, st.estimate, order_n, ctr)
    g = t_c + mm(r_c, nsp, ctr)
    f = I - mm(g, a, ctr)
    return NS(g, f, st.step + 1, order_n, st.series_order, ctr)


def initial_double(sp: Split, p: int, w: int, order: int = 2) -> DoubleNS:
    """ns:231-251."""
    base = initial_series(sp, p, w, order)
    l0 = _horner(base.residual, base.estimate, order, base.ctr)
    r0 = eye(l0.shape[0]) - mm(l0, sp.matrix, base.ctr)
    return DoubleNS(base.estimate, base.residual, l0, r0, 0, order, base.series_order, base.ctr)


def double_ns_step(st: DoubleNS, a) -> DoubleNS:
    """ns:254-298 (serial order: accelerator branch, then main branch)."""
    n = st.order
    I = eye(a.shape[0])
    gamma = I - mm(st.accel_estimate, a, st.ctr)
    l_new = _horner(gamma, st.accel_estimate, n, st.ctr)
    r_new = I - mm(l_new, a, st.ctr)
    nsp = _horner(st.residual, st.estimate, n, st.ctr)
    g = l_new + mm(r_new, nsp, st.ctr)
    f = I - mm(g, a, st.ctr)
    return DoubleNS(g, f, l_new, r_new, st.step + 1, n, st.series_order, st.ctr)


def additive_correction_step(z, g, a, p, ctr):
    """ns:301-325."""
    I = eye(a.shape[0])
    l_prev = I - mm(z, a, ctr)
    z_new = _horner(l_prev, z, p, ctr)
    f_prev = I - mm(g, a, ctr)
    return z_new, g + mm(f_prev, z_new, ctr)


# ---------------------------------------------------------------------------
# L5: Richardson (ri:42-189) and the plain update
# ---------------------------------------------------------------------------


@dataclass
class Rich:
    """ri:42-58."""

    theta: np.ndarray
    inner: DoubleNS
    q: int
    omega: np.ndarray | None
    ns_part: np.ndarray | None
    step: int
    ctr: Counter


def initial_richardson(sp: Split, b, p=0, w=1, order=2, q=None) -> Rich:
    """ri:61-78 -- theta_0 = L_0 b."""
    inner = initial_double(sp, p, w, order)
    q = order if q is None else q
    theta = mv(inner.accel_estimate, b, inner.ctr)
    return Rich(theta, inner, q, None, None, 0, inner.ctr)


def richardson_step(st: Rich, a, b) -> Rich:
    """ri:81-98."""
    inner = double_ns_step(st.inner, a)
    s = _horner(inner.residual, inner.estimate, st.q, st.ctr)
    wgt = inner.accel_estimate + mm(inner.accel_residual, s, st.ctr)
    resid = mv(a, st.theta, st.ctr) - b
    theta = st.theta - mv(wgt, resid, st.ctr)
    return Rich(theta, inner, st.q, None, None, st.step + 1, st.ctr)


def power_sum(gamma, n, ctr):
    """ri:101-108 -- I + gamma + ... + gamma^(n-1), n-2 products."""
    acc = eye(gamma.shape[0])
    cur = None
    for _ in range(n - 1):
        cur = gamma if cur is None else mm(cur, gamma, ctr)
        acc = acc + cur
    return acc


def richardson_recursive_step(st: Rich, a, b) -> Rich:
    """ri:111-189 (serial order: estimate part, then accel part)."""
    n = st.inner.order
    if st.q != n:
        raise ValueError("the recursive form requires q == n")
    prev = st.inner
    I = eye(a.shape[0])
    if st.omega is None or st.ns_part is None:
        ns_prev = _horner(prev.residual, prev.estimate, n, st.ctr)
        om_prev = prev.accel_estimate + mm(prev.accel_residual, ns_prev, st.ctr)
    else:
        ns_prev, om_prev = st.ns_part, st.omega
    s = power_sum(prev.accel_residual, n, st.ctr)
    g = mm(s, om_prev - ns_prev, st.ctr) + ns_prev
    f = I - mm(g, a, st.ctr)
    ns_new = _horner(f, g, n, st.ctr)
    l_new = mm(s, prev.accel_estimate, st.ctr)
    r_new = I - mm(l_new, a, st.ctr)
    om = l_new + mm(r_new, ns_new, st.ctr)
    resid = mv(a, st.theta, st.ctr) - b
    theta = st.theta - mv(om, resid, st.ctr)
    inner = DoubleNS(g, f, l_new, r_new, prev.step + 1, n, prev.series_order, st.ctr)
    return Rich(theta, inner, st.q, om, ns_new, st.step + 1, st.ctr)


def plain_richardson(theta, p, a, b, ctr):
    """theta + P (b - A theta), products through mat_vec exactly
    as ri:88-89: resid = A theta - b; theta - P resid."""
    resid = mv(a, theta, ctr) - b
    return theta - mv(p, resid, ctr)


def converged(residual) -> bool:
    """ns:328-331."""
    return fro(residual) <= 1e-13 * np.sqrt(residual.shape[0])
