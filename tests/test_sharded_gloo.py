"""Multi-rank block-row sharded steps on CPU: world_size 2 over gloo.

The orchestration (row splits, all-gathers of sharded right operands, shifted
diagonals, the composite fold) is the product code in
paper_2008_11480_b200/sharded.py; only the local-ops layer is swapped for a
CPU torch implementation here.  Results are compared with the oracle on the
same inputs, and the GEMM count with the reference DAG.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


class CpuOps:
    """Test-only local ops (CPU float64 torch)."""

    def gemm(self, a, b, alpha, c, beta, diag, doff, is_mv, ctr):
        out = alpha * (a @ b)
        if c is not None:
            out = out + beta * c
        if diag:
            rows = torch.arange(out.shape[0])
            cols = rows + doff
            ok = cols < out.shape[1]
            out[rows[ok], cols[ok]] += diag
        if is_mv:
            ctr.mvm += 1
        else:
            ctr.mmm += 1
        return out

    def sumsq(self, x):
        return float((x * x).sum())

    def lin(self, cdiag, doff, terms, rows, cols, like):
        out = torch.zeros((rows, cols), dtype=torch.float64)
        if cdiag:
            r = torch.arange(rows)
            ok = r + doff < cols
            out[r[ok], (r + doff)[ok]] = cdiag
        for coef, t in terms:
            out = out + coef * t
        return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir, n, steps):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200.sharded import RowComm, ShardedEngine

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    a_np, b_np = configs.c4_householder(n=n, rhs=3)
    alpha = np.max(np.sum(np.abs(a_np), axis=1))
    comm = RowComm(n)
    eng = ShardedEngine(comm, ops=CpuOps())
    A = eng.replicated(torch.as_tensor(a_np))
    P = eng.replicated(torch.eye(n, dtype=torch.float64) / alpha)
    B = eng.replicated(torch.eye(n, dtype=torch.float64) - torch.as_tensor(a_np) / alpha)
    b = eng.replicated(torch.as_tensor(b_np))
    g = eng.local(P.t[comm.r0:comm.r1].clone())
    f = eng.local(B.t[comm.r0:comm.r1].clone())
    theta = eng.replicated(torch.zeros_like(b.t))
    for _ in range(steps):
        theta = eng.plain_richardson(theta, g, A, b)
        g, f = eng.composite_step(g, f, A, P, B, (2, 3, 4, 5), 2)
    g_full = comm.all_gather_rows(g.t)
    f_norm = eng.fro_norm(f)           # one scalar all-reduce (stop rule)
    f_conv = eng.converged(f, n)
    h_full = eng.ns_step(g, f, A, 8, plan=None)[0]
    h_full = comm.all_gather_rows(h_full.t)
    if rank == 0:
        np.save(os.path.join(outdir, "g.npy"), g_full.numpy())
        np.save(os.path.join(outdir, "theta.npy"), theta.t.numpy())
        np.save(os.path.join(outdir, "h.npy"), h_full.numpy())
        np.save(os.path.join(outdir, "ctr.npy"), np.array([eng.ctr.mmm, eng.ctr.mvm]))
        np.save(os.path.join(outdir, "gathered.npy"), np.array([comm.bytes_gathered]))
        np.save(os.path.join(outdir, "fnorm.npy"), np.array([f_norm, float(f_conv)]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 41), (3, 24)])
def test_sharded_composite_matches_oracle(world, n):
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    steps = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, n, steps), nprocs=world, join=True)
        g = np.load(os.path.join(d, "g.npy"))
        theta = np.load(os.path.join(d, "theta.npy"))
        h = np.load(os.path.join(d, "h.npy"))
        ctr = np.load(os.path.join(d, "ctr.npy"))
        gathered = int(np.load(os.path.join(d, "gathered.npy"))[0])
        f_norm, f_conv = np.load(os.path.join(d, "fnorm.npy"))
    a, b = configs.c4_householder(n=n, rhs=3)
    sp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    st = O.initial_series(sp, 0, 1, 2)
    th = np.zeros_like(b)
    for _ in range(steps):
        th = O.plain_richardson(th, st.estimate, sp.matrix, b, st.ctr)
        st = O.composite_step(st, sp.matrix, sp, (2, 3, 4, 5), 2)
    mmm_ref, mvm_ref = st.ctr.mmm, st.ctr.mvm
    # ns_step with order 8 on the final state (Horner)
    st8 = O.NS(st.estimate, st.residual, st.step, 8, 1, O.Counter())
    h_ref = O.ns_step(st8, sp.matrix).estimate
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)  # noqa: E731
    assert rel(g, st.estimate) <= 1e-11
    assert rel(theta, th) <= 1e-11
    assert rel(h, h_ref) <= 1e-11
    # sharded ||F||_F (ns:328-331 stop rule) = the oracle's full-matrix norm
    f_ref = np.linalg.norm(st.residual)  # matrix_core.fro_norm (mc:167-168)
    assert abs(f_norm - f_ref) <= 1e-11 * f_ref
    assert bool(f_conv) == (f_ref <= 1e-13 * np.sqrt(n))
    # same DAG as the reference: 22 products + 2 per composite step, then 8 for ns_step(8)
    assert int(ctr[0]) == mmm_ref + 8 and int(ctr[1]) == mvm_ref
    assert gathered > 0


def _worker_recursive(rank, world, port, outdir, n, steps, factorised):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200.sharded import RowComm, ShardedEngine
    from paper_2008_11480_b200.series_toolkit import plan_order

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    a_np, b_np = _c5_like(n)
    # initial state from the oracle (initial_richardson is setup, not the sharded step)
    sp = O.split_scalar(a_np, O.inf_norm(a_np) / 2.0)
    st = O.initial_richardson(sp, b_np, 0, 1, 4, 4)
    comm = RowComm(n)
    eng = ShardedEngine(comm, ops=CpuOps())
    rows = slice(comm.r0, comm.r1)
    loc = lambda m: eng.local(torch.as_tensor(m[rows]).clone())  # noqa: E731
    g, f, l, r = (loc(m) for m in (st.inner.estimate, st.inner.residual,
                                    st.inner.accel_estimate, st.inner.accel_residual))
    A = eng.replicated(torch.as_tensor(sp.matrix))
    b = eng.replicated(torch.as_tensor(b_np))
    theta = eng.replicated(torch.as_tensor(st.theta))
    om = ns = None
    kw = {"factor_plan": plan_order(4), "doubling_sum": True} if factorised else {}
    for _ in range(steps):
        g, f, l, r, om, ns, theta = eng.richardson_recursive_step(g, f, l, r, om, ns, A, theta, b,
                                                                   4, **kw)
    g_full = comm.all_gather_rows(g.t)
    om_full = comm.all_gather_rows(om.t)
    if rank == 0:
        np.save(os.path.join(outdir, "g.npy"), g_full.numpy())
        np.save(os.path.join(outdir, "om.npy"), om_full.numpy())
        np.save(os.path.join(outdir, "theta.npy"), theta.t.numpy())
        np.save(os.path.join(outdir, "ctr.npy"), np.array([eng.ctr.mmm, eng.ctr.mvm]))
    dist.destroy_process_group()


def _c5_like(n):
    rng = np.random.default_rng(5)
    g = rng.standard_normal((n + n // 4, n))
    a = g.T @ g / (n + n // 4) + 1e-3 * np.eye(n)
    return (a + a.T) / 2.0, rng.standard_normal((n, 3))


@pytest.mark.parametrize("world,n,factorised", [(2, 29, False), (3, 24, True)])
def test_sharded_recursive_richardson_matches_oracle(world, n, factorised):
    from oracle import seriesinv_oracle as O

    steps = 3
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_recursive, args=(world, _free_port(), d, n, steps, factorised),
                 nprocs=world, join=True)
        g = np.load(os.path.join(d, "g.npy"))
        om = np.load(os.path.join(d, "om.npy"))
        theta = np.load(os.path.join(d, "theta.npy"))
        ctr = np.load(os.path.join(d, "ctr.npy"))
    a, b = _c5_like(n)
    sp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    st = O.initial_richardson(sp, b, 0, 1, 4, 4)
    m0 = st.ctr.mmm
    for _ in range(steps):
        st = O.richardson_recursive_step(st, sp.matrix, b)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)  # noqa: E731
    tol = 1e-9 if factorised else 1e-11  # factorised sums reassociate the series
    assert rel(g, st.inner.estimate) <= tol
    assert rel(om, st.omega) <= tol
    assert rel(theta, st.theta) <= tol
    if not factorised:
        assert int(ctr[0]) == st.ctr.mmm - m0  # same DAG as the reference: 3n+2, then 2n+2


def test_row_splits_cover():
    from paper_2008_11480_b200.sharded import row_splits

    for n in (1, 7, 64, 1000):
        for w in (1, 2, 3, 8):
            s = row_splits(n, w)
            assert s[0][0] == 0 and s[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
            assert max(r1 - r0 for r0, r1 in s) - min(r1 - r0 for r0, r1 in s) <= 1
