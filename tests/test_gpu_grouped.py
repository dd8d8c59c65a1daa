"""Composite parts on GPU groups (grouped.py) on the device path.

* one process: the single-group step is the library's composite_step bitwise
  (same products, same order inside the fold), 22 products per step;
* 2 and 4 processes sharing cuda:0 (gloo, the tree's (t, r) blocks staged
  through the host -- no kernel waits on another process): the DMMA products
  of every group against the oracle within the FP64 tolerance, and the product
  count summed over the groups equal to the reference DAG's.
"""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, release_gpu_memory
from test_sharded_gloo import _free_port

pytestmark = pytest.mark.gpu


def test_single_group_bitwise_vs_composite_step():
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200.grouped import GroupedComposite

    n = 384
    a, _ = configs.c4_householder(n=n, rhs=1)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0)
    st = P.initial_series(sp, 0, 1, order=2)
    gc = GroupedComposite(n, (2, 3, 4, 5), 2)
    eng = gc.eng
    g, f = eng.local(st.estimate.clone()), eng.local(st.residual.clone())
    A, Pm, B = (eng.replicated(x) for x in (sp.matrix, sp.precond, sp.residual))
    for _ in range(3):
        g, f = gc.step(g, f, A, Pm, B)
        st = P.composite_step(st, sp.matrix, sp, P.CompositeSpec((2, 3, 4, 5)), 2)
    torch.cuda.synchronize()
    assert torch.equal(g.t, st.estimate) and torch.equal(f.t, st.residual)
    assert gc.products_executed() == 66


def _worker(rank, world, port, outdir, n, steps):
    import sys

    sys.path.insert(0, ROOT)
    torch.cuda.set_device(0)
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200.grouped import GroupedComposite

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    a_np, b_np = configs.c4_householder(n=n, rhs=4)
    sp = P.split_scalar(a_np, P.inf_norm(a_np) / 2.0)
    st = P.initial_series(sp, 0, 1, order=2)
    gc = GroupedComposite(n, (2, 3, 4, 5), 2)
    eng, comm = gc.eng, gc.comm
    A, Pm, B = (eng.replicated(x) for x in (sp.matrix, sp.precond, sp.residual))
    b = eng.replicated(P.as_device(b_np))
    g = eng.local(st.estimate[comm.r0:comm.r1].clone())
    f = eng.local(st.residual[comm.r0:comm.r1].clone())
    theta = eng.replicated(torch.zeros_like(b.t))
    for _ in range(steps):
        theta = gc.plain_richardson(theta, g, A, b)
        g, f = gc.step(g, f, A, Pm, B)
    torch.cuda.synchronize()
    total = gc.products_executed()
    g_full = comm.all_gather_rows(g.t)
    f_full = comm.all_gather_rows(f.t)
    if rank == 0:
        np.save(os.path.join(outdir, "g.npy"), g_full.cpu().numpy())
        np.save(os.path.join(outdir, "f.npy"), f_full.cpu().numpy())
        np.save(os.path.join(outdir, "theta.npy"), theta.t.cpu().numpy())
        np.save(os.path.join(outdir, "meta.npy"), np.array([total, len(gc.groups)]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_grouped_processes_vs_oracle(world):
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    release_gpu_memory()
    n, steps = 256, 3
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, n, steps), nprocs=world, join=True)
        g = np.load(os.path.join(d, "g.npy"))
        f = np.load(os.path.join(d, "f.npy"))
        theta = np.load(os.path.join(d, "theta.npy"))
        total, ngroups = (int(x) for x in np.load(os.path.join(d, "meta.npy")))
    a, b = configs.c4_householder(n=n, rhs=4)
    sp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    st = O.initial_series(sp, 0, 1, 2)
    th = np.zeros_like(b)
    m0 = st.ctr.mmm
    for _ in range(steps):
        th = O.plain_richardson(th, st.estimate, sp.matrix, b, st.ctr)
        st = O.composite_step(st, sp.matrix, sp, (2, 3, 4, 5), 2)
    kappa = np.linalg.cond(a)
    tol = 1e-10 * max(1.0, kappa / 1e4)  # north_star tolerance, kappa-scaled
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)  # noqa: E731
    assert rel(g, st.estimate) <= tol
    assert rel(theta, th) <= tol
    assert np.linalg.norm(f - st.residual) / np.sqrt(n) <= tol
    assert total == st.ctr.mmm - m0 == 66
    assert ngroups == min(world, 4)
