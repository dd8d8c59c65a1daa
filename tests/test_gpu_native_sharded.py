"""Block-row sharded steps through the C ABI (si_comm_* / si_sharded_*,
SURVEY 8(b)/8(e)): the library orchestrates the row-sharded DAG and its
all-gathers, so a C / cgo / JNI host can run the multi-GPU path.

* world 1 with a real NCCL communicator (one GPU per box here): bitwise the
  single-GPU steps, same counters;
* 2 and 3 processes sharing cuda:0 with the host (gloo) exchange: every
  rank's row blocks, theta and the sharded stop-rule norm against the
  single-GPU steps -- bitwise, since the per-tile K order does not depend on
  the row split (n = 386: uneven blocks).
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _single_gpu(n):
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a_np, b_np = configs.c4_householder(n=n, rhs=3)
    a, b = P.as_device(a_np), P.as_device(b_np)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1, order=2)
    theta = torch.zeros_like(b)
    for _ in range(2):
        theta = P.plain_richardson(theta, st.estimate, sp.matrix, b, st.ctr)
        st = P.composite_step(st, sp.matrix, sp, P.CompositeSpec((2, 3, 4, 5)), 2)
    rs = P.initial_richardson(sp, b, 0, 1, order=4, q=4)
    c0 = rs.ctr.mmm, rs.ctr.mvm
    for _ in range(2):
        rs = P.richardson_recursive_step(rs, sp.matrix, b, factor_plan=P.plan_order(4),
                                         doubling_sum=True)
    return {"g": st.estimate.cpu().numpy(), "f": st.residual.cpu().numpy(),
            "theta": theta.cpu().numpy(), "fro": float(P.fro_norm(st.residual)),
            "ctr": (st.ctr.mmm, st.ctr.mvm), "rg": rs.inner.estimate.cpu().numpy(),
            "romega": rs.omega.cpu().numpy(), "rtheta": rs.theta.cpu().numpy(),
            "rctr": (rs.ctr.mmm - c0[0], rs.ctr.mvm - c0[1])}


def test_nccl_world_one_bitwise():
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200 import native_sharded as NS

    n = 512
    ref = _single_gpu(n)
    comm = NS.NativeComm.nccl(n)
    assert (comm.r0, comm.r1, comm.world) == (0, n, 1)
    a_np, b_np = configs.c4_householder(n=n, rhs=3)
    a, b = P.as_device(a_np), P.as_device(b_np)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1, order=2)
    ctr = P.MulCounter()
    g, f, theta = st.estimate, st.residual, torch.zeros_like(b)
    for _ in range(2):
        theta = NS.plain_richardson(comm, theta, g, sp.matrix, b, ctr)
        g, f = NS.composite_step(comm, g, f, sp.matrix, sp.precond, sp.residual, sp.matrix,
                                 (2, 3, 4, 5), 2, ctr)
    assert np.array_equal(g.cpu().numpy(), ref["g"])
    assert np.array_equal(f.cpu().numpy(), ref["f"])
    assert np.array_equal(theta.cpu().numpy(), ref["theta"])
    assert (ctr.mmm, ctr.mvm) == ref["ctr"]
    assert NS.fro_norm(comm, f) == pytest.approx(ref["fro"], rel=1e-14)
    # ns_step with the h8 plan
    st8 = P.initial_series(sp, 0, 1, order=8)
    want = P.ns_step(st8, sp.matrix, plan=P.table_plans()[8][0])
    g8, f8 = NS.ns_step(comm, st8.estimate, st8.residual, sp.matrix, 8, P.table_plans()[8][0])
    assert torch.equal(g8, want.estimate) and torch.equal(f8, want.residual)
    comm.close()


@pytest.mark.parametrize("backend", ["dmma", "ozaki"])
@pytest.mark.parametrize("world", [2, 3])
def test_processes_share_gpu_host_exchange(world, backend, tmp_path):
    """Block-row steps through si_sharded_* in `world` processes: bitwise the
    single-GPU steps -- also with every product emulated on the INT8 tensor
    cores (row splits change no bit: each row's scale and the integer
    products are its own)."""
    import paper_2008_11480_b200 as P
    from conftest import release_gpu_memory

    release_gpu_memory()
    n = 386
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native_shard_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), port, str(tmp_path),
                               str(n), backend]) for r in range(world)]
    try:
        codes = [p.wait(timeout=300) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert codes == [0] * world
    with P.gemm_backend(backend, moduli=16, min_dim=128):
        ref = _single_gpu(n)
    from paper_2008_11480_b200.sharded import row_splits

    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for key in ("g", "f", "rg", "romega"):
        assert np.array_equal(np.concatenate([p[key] for p in parts]), ref[key]), key
    for p, (r0, r1) in zip(parts, row_splits(n, world)):
        assert p[key].shape[0] == r1 - r0
        assert np.array_equal(p["theta"], ref["theta"])  # replicated on every rank
        assert np.array_equal(p["rtheta"], ref["rtheta"])
        assert float(p["fro"]) == pytest.approx(ref["fro"], rel=1e-13)
        c = p["ctr"]
        assert (c[0], c[1]) == ref["ctr"] and (c[2], c[3]) == ref["rctr"]
        assert c[4] > 0 and c[5] > 0  # gathers happened
