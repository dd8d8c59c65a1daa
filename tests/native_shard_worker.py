"""Worker of tests/test_gpu_native_sharded.py: one process per rank (all on
cuda:0), the block-row steps through the C ABI (si_sharded_*) with a host
exchange over gloo (no kernel waits on another process).  Writes this rank's
row blocks and counters to <out>/rank<r>.npz."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world, port, out, n = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4],
                                 int(sys.argv[5]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200 import native_sharded as NS

    if len(sys.argv) > 6 and sys.argv[6] == "ozaki":
        P.set_gemm_backend("ozaki", 16, 128)

    a_np, b_np = configs.c4_householder(n=n, rhs=3)
    a = P.as_device(a_np)
    b = P.as_device(b_np)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1, order=2)
    comm = NS.NativeComm.host(n)
    ctr = P.MulCounter()
    g, f = comm.rows_of(st.estimate), comm.rows_of(st.residual)
    theta = torch.zeros_like(b)
    for _ in range(2):
        theta = NS.plain_richardson(comm, theta, g, sp.matrix, b, ctr)
        g, f = NS.composite_step(comm, g, f, sp.matrix, sp.precond, sp.residual, sp.matrix,
                                 (2, 3, 4, 5), 2, ctr)
    fro = NS.fro_norm(comm, f)
    # recursive Richardson / factorised order 4 from the same splitting
    rs = P.initial_richardson(sp, b, 0, 1, order=4, q=4)
    inner = rs.inner
    state = [comm.rows_of(x) for x in (inner.estimate, inner.residual, inner.accel_estimate,
                                        inner.accel_residual)] + [None, None]
    th2 = rs.theta
    rctr = P.MulCounter()
    for _ in range(2):
        state, th2 = NS.richardson_recursive_step(comm, state, sp.matrix, th2, b, 4,
                                                  factor_plan=P.plan_order(4),
                                                  doubling_sum=True, ctr=rctr)
    torch.cuda.synchronize()
    gathers, nbytes = comm.stats()
    np.savez(os.path.join(out, f"rank{rank}.npz"), g=g.cpu().numpy(), f=f.cpu().numpy(),
             theta=theta.cpu().numpy(), fro=np.array(fro), rg=state[0].cpu().numpy(),
             romega=state[4].cpu().numpy(), rtheta=th2.cpu().numpy(),
             ctr=np.array([ctr.mmm, ctr.mvm, rctr.mmm, rctr.mvm, gathers, nbytes]))
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
