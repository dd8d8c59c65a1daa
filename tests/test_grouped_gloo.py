"""Composite parts on GPU groups + one ordered tree reduction, on CPU.

The orchestration (group/segment planning, per-group left folds, the ordered
(t, r) tree over point-to-point transfers, block-row sharding inside a group)
is the product code in paper_2008_11480_b200/grouped.py; only the local-ops
layer is the CPU one of test_sharded_gloo.py.  Compared with the oracle
(newton_schulz.py:177-228 restated) on the same inputs; the products summed
over the groups must equal the reference DAG's count.
"""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT
from test_sharded_gloo import CpuOps, _free_port


def test_part_costs_match_the_reference_dag():
    from paper_2008_11480_b200.grouped import part_cost

    # T_x via plan_order(x) (x <= 64) or doubling, plus Gamma = I - T A
    assert [part_cost(x) for x in (1, 2, 3, 4, 5)] == [1, 2, 3, 4, 4]
    assert part_cost(100) > part_cost(64)


def test_plan_groups_shapes():
    from paper_2008_11480_b200.grouped import plan_groups

    costs = [2, 3, 4, 4]
    for world in (1, 2, 3, 4, 8, 16):
        groups, segs = plan_groups(world, costs, 2)
        assert len(groups) == len(segs) == min(world, 4)
        assert sorted(r for g in groups for r in g) == list(range(world))
        assert [i for s in segs for i in s] == [0, 1, 2, 3]  # contiguous, ordered
        assert all(s for s in segs)
    assert plan_groups(2, costs, 2)[1] == [[0, 1], [2, 3]]
    assert plan_groups(8, costs, 2)[0] == [[0, 1], [2, 3], [4, 5], [6, 7]]
    with pytest.raises(ValueError):
        plan_groups(2, [], 2)


def _worker(rank, world, port, outdir, n, steps, rates, order_n=2):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200.grouped import GroupedComposite

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    a_np, b_np = configs.c4_householder(n=n, rhs=3)
    alpha = np.max(np.sum(np.abs(a_np), axis=1))
    gc = GroupedComposite(n, rates, order_n, ops=CpuOps())
    eng, comm = gc.eng, gc.comm
    A = eng.replicated(torch.as_tensor(a_np))
    P = eng.replicated(torch.eye(n, dtype=torch.float64) / alpha)
    B = eng.replicated(torch.eye(n, dtype=torch.float64) - torch.as_tensor(a_np) / alpha)
    b = eng.replicated(torch.as_tensor(b_np))
    g = eng.local(P.t[comm.r0:comm.r1].clone())
    f = eng.local(B.t[comm.r0:comm.r1].clone())
    theta = eng.replicated(torch.zeros_like(b.t))
    for _ in range(steps):
        theta = gc.plain_richardson(theta, g, A, b)
        g, f = gc.step(g, f, A, P, B)
    total = gc.products_executed()
    g_full = comm.all_gather_rows(g.t)
    f_full = comm.all_gather_rows(f.t)
    if rank == 0:
        np.save(os.path.join(outdir, "g.npy"), g_full.numpy())
        np.save(os.path.join(outdir, "f.npy"), f_full.numpy())
        np.save(os.path.join(outdir, "theta.npy"), theta.t.numpy())
        np.save(os.path.join(outdir, "meta.npy"),
                np.array([total, len(gc.groups), gc.ctr.mvm]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,rates,order_n", [
    (2, 40, (2, 3, 4, 5), 2), (4, 33, (2, 3, 4, 5), 2), (3, 24, (2, 3, 1, 4, 5), 2),
    (5, 26, (2, 3, 4, 5), 2), (8, 40, (2, 3, 4, 5), 2), (6, 30, (2, 3, 4), 2),
    (2, 21, (3, 2), 1), (3, 27, (2, 5, 3), 3)])
def test_grouped_composite_matches_oracle(world, n, rates, order_n):
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    steps = 3
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, n, steps, rates, order_n), nprocs=world,
                 join=True)
        g = np.load(os.path.join(d, "g.npy"))
        f = np.load(os.path.join(d, "f.npy"))
        theta = np.load(os.path.join(d, "theta.npy"))
        total, ngroups, mvm = (int(x) for x in np.load(os.path.join(d, "meta.npy")))
    a, b = configs.c4_householder(n=n, rhs=3)
    sp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    st = O.initial_series(sp, 0, 1, 2)
    th = np.zeros_like(b)
    m0 = st.ctr.mmm
    for _ in range(steps):
        th = O.plain_richardson(th, st.estimate, sp.matrix, b, st.ctr)
        st = O.composite_step(st, sp.matrix, sp, rates, order_n)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)  # noqa: E731
    # the tree associates the fold differently: rounding-level, kappa-scaled
    assert rel(g, st.estimate) <= 1e-10
    assert rel(theta, th) <= 1e-10
    assert np.linalg.norm(f - st.residual) / np.sqrt(n) <= 1e-10
    # same number of products as the reference DAG, summed over the groups
    assert total == st.ctr.mmm - m0
    assert ngroups == min(world, len(rates))
    assert mvm == st.ctr.mvm


def test_single_group_is_the_reference_fold_bitwise():
    """No process group: one group, the left fold of newton_schulz.py:212-216."""
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200.grouped import GroupedComposite
    from paper_2008_11480_b200.sharded import RowComm, ShardedEngine

    n = 20
    a_np, _ = configs.c4_householder(n=n, rhs=1)
    alpha = np.max(np.sum(np.abs(a_np), axis=1))
    gc = GroupedComposite(n, (2, 3, 4, 5), 2, ops=CpuOps())
    ref = ShardedEngine(RowComm(n), ops=CpuOps())
    A = torch.as_tensor(a_np)
    P = torch.eye(n, dtype=torch.float64) / alpha
    B = torch.eye(n, dtype=torch.float64) - A / alpha
    outs = []
    for eng, fn in ((gc.eng, gc.step), (ref, lambda g, f, a, p, r: ref.composite_step(
            g, f, a, p, r, (2, 3, 4, 5), 2))):
        g, f = eng.local(P.clone()), eng.local(B.clone())
        for _ in range(2):
            g, f = fn(g, f, eng.replicated(A), eng.replicated(P), eng.replicated(B))
        outs.append((g.t, f.t, eng.ctr.mmm if eng is ref else gc.ctr.mmm))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2] == 44
    assert gc.ctr.mmm == 44
