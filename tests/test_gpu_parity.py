"""CUDA path vs the reference (golden fixtures) and the CPU oracle, through the C ABI.

Tolerance (SURVEY 8c / BASELINE.json north_star): relative Frobenius error of
P_k and theta_k <= 1e-10 * max(1, kappa(A)/1e4); residual-like matrices
(F = I - G A, which converge to 0) use ||dF||_F / sqrt(n) <= 1e-10.
Integer MulCounter deltas must match the reference exactly.
"""

import numpy as np
import pytest
import torch

import cases
from conftest import golden

pytestmark = pytest.mark.gpu

TOL = 1e-10


def kappa_tol(a):
    ev = np.linalg.eigvalsh((a + a.T) / 2.0)
    kappa = float(ev.max() / ev.min())
    return TOL * max(1.0, kappa / 1e4)


@pytest.fixture(scope="module")
def B():
    from gpu_backend import GpuBackend

    return GpuBackend()


@pytest.fixture(scope="module")
def Bc():
    from gpu_backend import GpuBackend

    return GpuBackend(concurrent=True)


def test_native_library_is_loaded(B):
    from paper_2008_11480_b200 import _lib

    assert torch.cuda.is_available()
    _lib.handle()
    assert _lib._lib is not None and _lib._lib._name.endswith("libseriesinv_b200.so")


# ---------------------------------------------------------------- GEMM seam

GEMM_SHAPES = [
    (1, 1, 1), (2, 3, 4), (5, 5, 5), (7, 5, 3), (64, 64, 64), (65, 63, 61), (128, 128, 128),
    (130, 70, 300), (257, 129, 511), (512, 512, 512), (1000, 1000, 1000), (384, 64, 384),
    (256, 256, 1), (300, 2, 300), (1024, 4, 1024), (2048, 2048, 2048),
]


@pytest.mark.parametrize("m,n,k", GEMM_SHAPES)
@pytest.mark.parametrize("epi", ["plain", "residual", "addc", "subc"])
def test_gemm_epilogues_vs_numpy(m, n, k, epi):
    from paper_2008_11480_b200 import _lib

    rng = np.random.default_rng(m * 7919 + n * 31 + k)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    c = rng.standard_normal((m, n))
    alpha, beta, diag = {"plain": (1.0, 0.0, 0.0), "residual": (-1.0, 0.0, 1.0),
                         "addc": (1.0, 1.0, 0.0), "subc": (-1.0, 1.0, 0.0)}[epi]
    ref = alpha * (a @ b) + beta * c + diag * np.eye(m, n)
    ta, tb, tc = (torch.as_tensor(x, device="cuda") for x in (a, b, c))
    td = torch.empty((m, n), dtype=torch.float64, device="cuda")
    buf = _lib.counter_buf()
    _lib.call("si_gemm", _lib.handle(), m, n, k, alpha, ta.data_ptr(), k, tb.data_ptr(), n, beta,
              tc.data_ptr() if beta else None, n, diag, td.data_ptr(), n, 0, buf, _lib.stream_ptr())
    out = td.cpu().numpy()
    # entrywise bound of one FP64 dot product of length k
    bound = 4 * k * np.finfo(float).eps * (np.abs(a) @ np.abs(b)) + 4 * np.finfo(float).eps * np.abs(c) + 1e-300
    assert np.all(np.abs(out - ref) <= bound + 1e-15), f"max err {np.max(np.abs(out - ref))}"
    assert buf[0] == 1 and buf[1] == 0


def test_gemm_strided_and_inplace():
    from paper_2008_11480_b200 import _lib

    rng = np.random.default_rng(5)
    big = torch.as_tensor(rng.standard_normal((300, 400)), device="cuda")
    a = big[:200, :150]           # lda = 400
    b = big[100:250, 200:390]     # ldb = 400, odd offsets
    c = torch.as_tensor(rng.standard_normal((200, 190)), device="cuda")
    ref = a.cpu().numpy() @ b.cpu().numpy() + c.cpu().numpy()
    _lib.call("si_gemm", _lib.handle(), 200, 190, 150, 1.0, a.data_ptr(), 400, b.data_ptr(), 400,
              1.0, c.data_ptr(), 190, 0.0, c.data_ptr(), 190, 0, None, _lib.stream_ptr())
    assert np.allclose(c.cpu().numpy(), ref, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- golden parity


@pytest.mark.parametrize("name,fixture", [
    ("toolkit", "toolkit.npz"), ("ns", "ns.npz"), ("richardson", "richardson.npz"),
    ("c1", "c1.npz"), ("c3", "c3.npz"), ("c4", "c4.npz"), ("c5", "c5.npz"),
])
def test_gpu_matches_reference_fixtures(B, name, fixture):
    g = golden(fixture)
    tol = kappa_tol(g["a"]) if g["a"].shape[0] >= 32 else TOL
    out = getattr(cases, f"case_{name}")(B)
    worst = cases.compare(out, fixture, B, rtol=tol, ftol=TOL)
    print(f"{fixture}: worst relative error {worst:.3e} (tol {tol:.1e})")


@pytest.mark.parametrize("name", ["c1", "c3", "c4", "c5"])
def test_gpu_matches_oracle_live(B, name):
    """Same seeded inputs through the live oracle (not only the stored fixture)."""
    ob = cases.OracleBackend()
    ref = getattr(cases, f"case_{name}")(ob)
    out = getattr(cases, f"case_{name}")(B)
    tol = kappa_tol(golden(f"{name}.npz")["a"])
    for key, val in ref.items():
        if isinstance(val, (int, np.integer)):
            assert int(out[key]) == int(val), key
            continue
        v = B.np(out[key])
        den = max(np.linalg.norm(val), 1e-300)
        assert np.linalg.norm(v - val) / den <= tol, key


# ---------------------------------------------------------------- executor mapping


def _bits(B, st_fields):
    return [B.np(x).tobytes() for x in st_fields]


def test_concurrent_streams_bitwise_equal_serial(B, Bc):
    g = golden("ns.npz")
    for backend_pair in ((B, Bc),):
        outs = []
        for be in backend_pair:
            a = be.dev(g["a"])
            sp = be.split_diagonal(a)
            st = be.initial_series(sp, 0, 1, 2)
            for _ in range(2):
                st = be.composite_step(st, sp.matrix, sp, (2, 3, 4, 5), 2)
            dst = be.initial_double(sp, 1, 2, 3)
            for _ in range(3):
                dst = be.double_ns_step(dst, sp.matrix)
            outs.append(_bits(be, [st.estimate, st.residual, dst.estimate, dst.accel_estimate])
                        + [st.ctr.mmm, dst.ctr.mmm])
        assert outs[0] == outs[1]
    gr = golden("richardson.npz")
    res = []
    for be in (B, Bc):
        a = be.dev(gr["a"])
        sp = be.split_scalar(a, 1.0 - be.inf_norm(a) / 2.0)
        st = be.initial_richardson(sp, be.dev(gr["b"]), 1, 2, 2, 2)
        for _ in range(3):
            st = be.richardson_recursive_step(st, sp.matrix, be.dev(gr["b"]))
        res.append(_bits(be, [st.theta, st.omega]) + [st.ctr.mmm])
    assert res[0] == res[1]


def test_concurrent_bitwise_at_size():
    """Serial vs concurrent composite step at n=1024 (multi-CTA GEMMs on two streams)."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a, _ = configs.c4_householder(n=1024, rhs=1)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    s1 = P.initial_series(sp, 0, 1, order=2)
    s2 = P.initial_series(sp, 0, 1, order=2)
    s1 = P.composite_step(s1, sp.matrix, sp, P.CompositeSpec((2, 3, 4, 5)), 2)
    s2 = P.composite_step(s2, sp.matrix, sp, P.CompositeSpec((2, 3, 4, 5)), 2, executor=True)
    assert torch.equal(s1.estimate, s2.estimate) and torch.equal(s1.residual, s2.residual)
    assert s1.ctr.mmm == s2.ctr.mmm == 22


def test_sharded_engine_single_rank_bitwise_equals_native():
    """The block-row engine at world size 1 runs the same kernels on the same operands as
    the native composite step: results must be bitwise identical, counters equal."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200.sharded import RowComm, ShardedEngine

    a, b = configs.c4_householder(n=512, rhs=8)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    st = P.initial_series(sp, 0, 1, order=2)
    bd = P.as_device(b)
    theta = torch.zeros_like(bd)
    eng = ShardedEngine(RowComm(512))
    g, f = eng.local(st.estimate.clone()), eng.local(st.residual.clone())
    th = eng.replicated(theta.clone())
    A, Pc, B, bv = (eng.replicated(x) for x in (sp.matrix, sp.precond, sp.residual, bd))
    for _ in range(2):
        theta = P.plain_richardson(theta, st.estimate, sp.matrix, bd, st.ctr)
        st = P.composite_step(st, sp.matrix, sp, P.CompositeSpec((2, 3, 4, 5)), 2)
        th = eng.plain_richardson(th, g, A, bv)
        g, f = eng.composite_step(g, f, A, Pc, B, (2, 3, 4, 5), 2)
    assert torch.equal(g.t, st.estimate) and torch.equal(f.t, st.residual)
    assert torch.equal(th.t, theta)
    assert (eng.ctr.mmm, eng.ctr.mvm) == (st.ctr.mmm - 0, st.ctr.mvm)


# ---------------------------------------------------------------- batched (config 2)


def test_batched_matches_reference_per_iteration(B):
    import paper_2008_11480_b200 as P

    g = golden("c2.npz")
    a = torch.as_tensor(g["a"], device="cuda")
    b = torch.as_tensor(g["b"], device="cuda")
    precond, residual = P.batched_scalar_split(a)
    p, f = precond.clone(), residual.clone()
    theta = torch.zeros_like(b)
    ctr = P.MulCounter()
    for k in range(1, 51):
        p, f, theta = P.batched_composite_richardson(a, b, precond, residual, p, f, theta, (2, 3), 2,
                                                     1, ctr)
        for i in range(a.shape[0]):
            ref = g[f"s{i}_theta_{k}"]
            err = np.linalg.norm(theta[i].cpu().numpy() - ref) / np.linalg.norm(ref)
            assert err <= TOL, (k, i, err)
            if f"s{i}_p_{k}" in g.files:
                refp = g[f"s{i}_p_{k}"]
                errp = np.linalg.norm(p[i].cpu().numpy() - refp) / np.linalg.norm(refp)
                assert errp <= TOL, (k, i, errp)
    assert ctr.mmm == int(g["s0_mmm"]) and ctr.mvm == int(g["s0_mvm"])


def test_batched_fused_iterations_equal_stepwise():
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a_np, b_np = configs.c2_batched(batch=300)
    a = torch.as_tensor(a_np, device="cuda")
    b = torch.as_tensor(b_np, device="cuda")
    precond, residual = P.batched_scalar_split(a)
    theta0 = torch.zeros_like(b)
    p1, f1, t1 = P.batched_composite_richardson(a, b, precond, residual, precond, residual, theta0,
                                                (2, 3), 2, 7)
    p2, f2, t2 = precond, residual, theta0
    for _ in range(7):
        p2, f2, t2 = P.batched_composite_richardson(a, b, precond, residual, p2, f2, t2, (2, 3), 2, 1)
    assert torch.equal(p1, p2) and torch.equal(f1, f2) and torch.equal(t1, t2)


def test_batched_odd_sizes_and_rates_vs_oracle():
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as o

    rng = np.random.default_rng(9)
    for n, rates, order_n in ((5, (2, 3), 2), (17, (1, 4, 5), 3), (32, (7,), 2)):
        batch = 6
        g = rng.standard_normal((batch, 2 * n, n))
        a_np = np.einsum("bki,bkj->bij", g, g) / (2 * n) + 0.1 * np.eye(n)
        b_np = rng.standard_normal((batch, n))
        a = torch.as_tensor(a_np, device="cuda")
        b = torch.as_tensor(b_np, device="cuda")
        precond, residual = P.batched_scalar_split(a)
        p, f, th = P.batched_composite_richardson(a, b, precond, residual, precond, residual,
                                                  torch.zeros_like(b), rates, order_n, 3)
        for i in range(batch):
            sp = o.split_scalar(a_np[i], o.inf_norm(a_np[i]) / 2.0)
            st = o.initial_series(sp, 0, 1, order_n)
            theta = np.zeros(n)
            for _ in range(3):
                theta = o.plain_richardson(theta, st.estimate, sp.matrix, b_np[i], st.ctr)
                st = o.composite_step(st, sp.matrix, sp, rates, order_n)
            assert np.linalg.norm(p[i].cpu().numpy() - st.estimate) <= TOL * np.linalg.norm(st.estimate)
            assert np.linalg.norm(th[i].cpu().numpy() - theta) <= TOL * np.linalg.norm(theta)


# ---------------------------------------------------------------- errors and purity


def test_reference_errors(B):
    import paper_2008_11480_b200 as P

    g = golden("ns.npz")
    sp = P.split_diagonal(g["a"])
    st = P.initial_series(sp, 0, 1, order=3)
    with pytest.raises(ValueError):
        P.ns_step(st, sp.matrix, plan=P.plan_order(4))
    with pytest.raises(ValueError):
        P.composite_step(st, sp.matrix, sp, P.CompositeSpec((2,)), 0)
    with pytest.raises(ValueError):
        P.ns_step(st, torch.eye(4, dtype=torch.float64, device="cuda"))
    rs = P.initial_richardson(sp, np.ones(5), order=2, q=3)
    with pytest.raises(ValueError):
        P.richardson_recursive_step(rs, sp.matrix, np.ones(5))
    x = sp.precond
    with pytest.raises(ValueError):
        P.horner_eval(sp.residual + 0.5, x, 3, P.MulCounter(), a=sp.matrix, form_y=True)
    with pytest.raises(ValueError):
        P.mat_mul(torch.eye(2, device="cuda", dtype=torch.float64),
                  torch.eye(3, device="cuda", dtype=torch.float64), P.MulCounter())


def test_inputs_never_mutated(B):
    import paper_2008_11480_b200 as P

    g = golden("ns.npz")
    sp = P.split_diagonal(g["a"])
    st = P.initial_double(sp, 1, 2, order=3)
    before = [x.clone() for x in (st.estimate, st.residual, st.accel_estimate, st.accel_residual,
                                  sp.matrix)]
    P.double_ns_step(st, sp.matrix)
    after = (st.estimate, st.residual, st.accel_estimate, st.accel_residual, sp.matrix)
    assert all(torch.equal(x, y) for x, y in zip(before, after))


# ---------------------------------------------------------------- full-size properties


def _row_sample_check(prod, a, b, rows, c=None, alpha=1.0, diag=0.0):
    """Check sampled rows of prod = alpha a@b + c + diag I against numpy."""
    an = a[rows].cpu().numpy()
    bn = b.cpu().numpy()
    ref = alpha * (an @ bn)
    if c is not None:
        ref = ref + c[rows].cpu().numpy()
    if diag:
        ref[np.arange(len(rows)), rows] += diag
    got = prod[rows].cpu().numpy()
    bound = 4 * a.shape[1] * np.finfo(float).eps * (np.abs(an) @ np.abs(bn)) + 1e-300
    assert np.all(np.abs(got - ref) <= bound + 1e-15)


@pytest.mark.parametrize("n", [4096, 8192])
def test_full_size_gemm_row_sampled(n):
    import paper_2008_11480_b200 as P

    torch.manual_seed(n)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    ctr = P.MulCounter()
    d = P.mat_mul(a, b, ctr)
    rows = np.random.default_rng(n).choice(n, 24, replace=False)
    _row_sample_check(d, a, b, rows)
    assert ctr.mmm == 1


def test_c4_full_size_step():
    """BASELINE config 4 at its full size (n=16384, 64 RHS): one composite step through
    the native engine equals the block-row engine bitwise (two independent
    orchestrations of the same DAG), F' = I - G' A holds on sampled rows, and the
    counters follow the reference DAG (22 mmm + 2 mvm)."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200.sharded import RowComm, ShardedEngine

    n = 16384
    a, b = configs.c4_householder_device(n=n, rhs=64)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    del a
    st = P.initial_series(sp, 0, 1, order=2)
    theta = torch.zeros_like(b)
    c0 = st.ctr.copy()
    theta1 = P.plain_richardson(theta, st.estimate, sp.matrix, b, st.ctr)
    st1 = P.composite_step(st, sp.matrix, sp, P.CompositeSpec((2, 3, 4, 5)), 2)
    assert (st1.ctr.mmm - c0.mmm, st1.ctr.mvm - c0.mvm) == (22, 2)
    eng = ShardedEngine(RowComm(n))
    A, Pc, B = (eng.replicated(x) for x in (sp.matrix, sp.precond, sp.residual))
    g, f = eng.composite_step(eng.local(st.estimate), eng.local(st.residual), A, Pc, B,
                              (2, 3, 4, 5), 2)
    th = eng.plain_richardson(eng.replicated(theta), eng.local(st.estimate), A, eng.replicated(b))
    assert torch.equal(g.t, st1.estimate) and torch.equal(f.t, st1.residual)
    assert torch.equal(th.t, theta1)
    rows = np.random.default_rng(4).choice(n, 8, replace=False)
    _row_sample_check(st1.residual, st1.estimate, sp.matrix, rows, alpha=-1.0, diag=1.0)
    # exponent law at full size: F_1 = B^(2+3+4+5) F_0^2 = B^16 since
    # F_0 = B; rows of B^16 by 15 row-vector products (checker: torch/cuBLAS)
    x = sp.residual[rows].clone()
    for _ in range(15):
        x = x @ sp.residual
    err = float(torch.linalg.norm(st1.residual[rows] - x) / torch.linalg.norm(x))
    assert err <= 1e-12, err


def test_c5_full_size_recursive_step():
    """BASELINE config 5 at its full size (n=32768, 256 RHS) through the opt-in
    factorised recursive step (the bench path), one steady-state step: 18
    products, F' = I - G' A on sampled rows, and the Richardson mismatch drops.
    The carried state is built from the splitting (G = L = omega = N = S^-1,
    F = R = B = I - S^-1 A, a consistent order-1 state) so the test runs the
    steady-state DAG without the 34 products of initial_richardson + the first
    call (oracle parity of the full 20-iteration run is at n=4096,
    test_gpu_fullsize.py)."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    n = 32768
    a, b = configs.c5_gram_device(n=n, m=40000, rhs=256)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    del a
    pre, res = sp.precond, sp.residual
    ctr = P.MulCounter()
    inner = P.DoubleNsState(estimate=pre, residual=res, accel_estimate=pre, accel_residual=res,
                            step=1, order=16, series_order=1, ctr=ctr)
    theta = torch.zeros_like(b)
    st = P.RichardsonState(theta=theta, inner=inner, q=16, omega=pre, ns_part=pre, step=1, ctr=ctr)
    r0 = float(torch.linalg.norm(b))  # A theta_0 - b with theta_0 = 0
    st1 = P.richardson_recursive_step(st, sp.matrix, b, factor_plan=P.plan_order(16),
                                      doubling_sum=True)
    assert (ctr.mmm, ctr.mvm) == (18, 2)
    r1 = float(torch.linalg.norm(sp.matrix @ st1.theta - b))
    assert r1 < r0
    rows = np.random.default_rng(5).choice(n, 4, replace=False)
    g = st1.inner.estimate
    f = st1.inner.residual
    x = (-(g[rows] @ sp.matrix)).cpu().numpy()
    x[np.arange(len(rows)), rows] += 1.0
    got = f[rows].cpu().numpy()
    assert np.max(np.abs(got - x)) <= 1e-9 * max(1.0, np.max(np.abs(x)))
    del st, st1, sp, g, f, b, inner, pre, res
    from conftest import release_gpu_memory

    release_gpu_memory()


def test_c3_full_size_properties():
    """BASELINE config 3 at n=4096: every step keeps F = I - G A (row-sampled) and the
    Richardson mismatch contracts; counters follow the reference DAG (6 mmm + 2 mvm)."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a_np, b_np = configs.c3_gram(n=4096)
    sp = P.split_scalar(a_np, P.inf_norm(a_np) / 2.0, check_pd=False)
    b = P.as_device(b_np)
    st = P.initial_series(sp, 0, 1, order=8)
    theta = torch.zeros_like(b)
    plan = P.table_plans()[8][0]
    rows = np.random.default_rng(3).choice(4096, 16, replace=False)
    norms = []
    for k in range(6):
        c0 = st.ctr.copy()
        theta = P.plain_richardson(theta, st.estimate, sp.matrix, b, st.ctr)
        f_prev = st.residual
        st = P.ns_step(st, sp.matrix, plan=plan)
        if k < 2:  # exponent law F_k = F_{k-1}^8 (ns:150-174), sampled rows
            x = f_prev[rows].clone()
            for _ in range(7):
                x = x @ f_prev
            err = float(torch.linalg.norm(st.residual[rows] - x) / torch.linalg.norm(x))
            assert err <= 1e-11, (k, err)
        assert (st.ctr.mmm - c0.mmm, st.ctr.mvm - c0.mvm) == (6, 2)
        _row_sample_check(st.residual, st.estimate, sp.matrix, rows, alpha=-1.0, diag=1.0)
        norms.append(float(torch.linalg.norm(sp.matrix @ theta - b)))
    assert all(n2 < n1 for n1, n2 in zip(norms, norms[1:]) if n1 > 1e-9)
    assert P.converged(st)


def test_resident_c1_matches_reference_per_iteration():
    """BASELINE config 1 through the resident kernel (state in shared memory)."""
    import paper_2008_11480_b200 as P

    g = golden("c1.npz")
    a = torch.as_tensor(g["a"], device="cuda")
    b = torch.as_tensor(g["b"], device="cuda")
    alpha = float(np.max(np.sum(np.abs(g["a"]), axis=1)))
    eye = torch.eye(64, dtype=torch.float64, device="cuda")
    p, f = eye / alpha, eye - a / alpha
    theta = torch.zeros_like(b)
    ctr = P.MulCounter()
    for k in range(1, 31):
        p, f, theta = P.batched_ns_richardson(a, b, p, f, theta, 3, 1, ctr=ctr)
        assert np.linalg.norm(theta.cpu().numpy() - g[f"theta_{k}"]) <= TOL * np.linalg.norm(g[f"theta_{k}"])
        assert np.linalg.norm(p.cpu().numpy() - g[f"p_{k}"]) <= TOL * np.linalg.norm(g[f"p_{k}"])
    assert (ctr.mmm, ctr.mvm) == (int(g["mmm"]), int(g["mvm"]))
    # one fused launch of all 30 iterations is bitwise the stepwise result
    p30, f30, t30 = P.batched_ns_richardson(a, b, eye / alpha, eye - a / alpha,
                                            torch.zeros_like(b), 3, 30)
    assert torch.equal(p30, p) and torch.equal(t30, theta)


def test_resident_ns_plan_and_batch_vs_oracle():
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as o

    rng = np.random.default_rng(11)
    batch, n = 5, 48
    g = rng.standard_normal((batch, 2 * n, n))
    a_np = np.einsum("bki,bkj->bij", g, g) / (2 * n) + 0.2 * np.eye(n)
    b_np = rng.standard_normal((batch, n))
    a = torch.as_tensor(a_np, device="cuda")
    b = torch.as_tensor(b_np, device="cuda")
    pre, res = P.batched_scalar_split(a)
    plan = P.table_plans()[8][0]
    p, f, th = P.batched_ns_richardson(a, b, pre, res, torch.zeros_like(b), 8, 4, plan=plan)
    for i in range(batch):
        sp = o.split_scalar(a_np[i], o.inf_norm(a_np[i]) / 2.0)
        st = o.initial_series(sp, 0, 1, 8)
        theta = np.zeros(n)
        for _ in range(4):
            theta = o.plain_richardson(theta, st.estimate, sp.matrix, b_np[i], st.ctr)
            st = o.ns_step(st, sp.matrix, o.TABLE_ROOTS[8][0][1])
        assert np.linalg.norm(p[i].cpu().numpy() - st.estimate) <= TOL * np.linalg.norm(st.estimate)
        assert np.linalg.norm(th[i].cpu().numpy() - theta) <= TOL * np.linalg.norm(theta)


@pytest.mark.parametrize("batch,n,cluster", [(64, 48, None), (40, 64, None), (5, 64, "2"),
                                             (5, 48, "8"), (3, 64, "0")])
def test_resident_ns_single_cta_and_cluster_sizes(batch, n, cluster, monkeypatch):
    """Config-1-shaped runs through both resident kernels: many systems (one CTA
    per system, 16 warps) and the cluster kernel with 2 / 8 CTAs per system (and
    cluster mode switched off), each vs the oracle per system."""
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as o

    if cluster is not None:
        monkeypatch.setenv("SI_RESIDENT_CLUSTER", cluster)
    rng = np.random.default_rng(batch * 1000 + n)
    g = rng.standard_normal((batch, 2 * n, n))
    a_np = np.einsum("bki,bkj->bij", g, g) / (2 * n) + 0.3 * np.eye(n)
    b_np = rng.standard_normal((batch, n))
    a = torch.as_tensor(a_np, device="cuda")
    b = torch.as_tensor(b_np, device="cuda")
    pre, res = P.batched_scalar_split(a)
    iters = 4
    p, f, th = P.batched_ns_richardson(a, b, pre, res, torch.zeros_like(b), 3, iters)
    for i in sorted({0, batch // 2, batch - 1}):
        sp = o.split_scalar(a_np[i], o.inf_norm(a_np[i]) / 2.0)
        st = o.initial_series(sp, 0, 1, 3)
        theta = np.zeros(n)
        for _ in range(iters):
            theta = o.plain_richardson(theta, st.estimate, sp.matrix, b_np[i], st.ctr)
            st = o.ns_step(st, sp.matrix)
        assert np.linalg.norm(p[i].cpu().numpy() - st.estimate) <= TOL * np.linalg.norm(st.estimate)
        assert np.linalg.norm(th[i].cpu().numpy() - theta) <= TOL * np.linalg.norm(theta)
