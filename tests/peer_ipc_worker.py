"""Worker of tests/test_gpu_peer.py::test_ipc_processes_composite_step: one
process per rank (both on cuda:0), gloo for the handle exchange, the block-row
composite step over PeerComm + IpcFabric in mode "stream" (no kernel waits on
another process), row blocks written to <out>/rank<r>.npy."""

import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world, port, out, n = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4],
                                 int(sys.argv[5]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200.peer import IpcFabric, PeerComm
    from paper_2008_11480_b200.sharded import ShardedEngine

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    g = rng.standard_normal((2 * n, n))
    a = torch.as_tensor(g.T @ g / (2 * n) + 0.5 * np.eye(n), device=dev)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1, order=2)
    comm = PeerComm(n, IpcFabric(dev), mode="stream")
    eng = ShardedEngine(comm)
    A, Pm, B = eng.replicated(a), eng.replicated(sp.precond), eng.replicated(sp.residual)
    gr = eng.local(st.estimate[comm.r0:comm.r1].clone())
    fr = eng.local(st.residual[comm.r0:comm.r1].clone())
    for _ in range(3):
        gr, fr = eng.composite_step(gr, fr, A, Pm, B, (2, 3, 4, 5), 2)
    torch.cuda.synchronize()
    np.save(os.path.join(out, f"rank{rank}.npy"),
            np.concatenate([eng.rows_of(gr).cpu().numpy(), eng.rows_of(fr).cpu().numpy()]))
    np.save(os.path.join(out, f"ctr{rank}.npy"), np.array([eng.ctr.mmm, len(comm._slots)]))
    del gr, fr, A, Pm, B
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
