"""Compute-only projection of the C-ABI block-row sharded C4 step
(si_sharded_composite_step) on one GPU: rank 0 of P ranks with an exchange
callback that fills the gathered buffer on the device (rank 0's own block
copied into every slot -- finite data, no host or NVLink traffic), timed for
P = 1, 2, 4, 8 on the chosen product backend.  A projection, not a multi-GPU
measurement: the real exchange adds (n - n/P) n 8 bytes per gathered operand.

    python tools/native_projection.py [--gemm ozaki|dmma] [--n 16384]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import _lib, configs  # noqa: E402
from paper_2008_11480_b200 import native_sharded as NS  # noqa: E402


def projection_comm(n, world, dev):
    h = _lib.handle(dev.index)

    def allgather(_ctx, send, recv, count, stream):
        for r in range(world):
            _lib.call("si_copy_async", h, recv + r * count * 8, send, count * 8, stream)
        return 0

    def allreduce(_ctx, buf, count, stream):
        return 0

    ag, ar = NS._AG(allgather), NS._AR(allreduce)
    out = ctypes.c_void_p()
    _lib.call("si_comm_create_callback", world, 0, n, ag, ar, None, ctypes.byref(out))
    return NS.NativeComm(out.value, n, 0, world, dev, keep=(ag, ar))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gemm", default="ozaki", choices=["ozaki", "dmma"])
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    n = args.n
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    a, b = configs.c4_householder_device(n=n, rhs=64)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    del a
    st = P.initial_series(sp, 0, 1, order=2)
    P.set_gemm_backend(args.gemm, 16, 1024)
    out = {"n": n, "gemm": args.gemm, "steps": args.steps,
           "note": "rank 0's share of si_sharded_composite_step; exchange = on-device copies"}
    base = None
    for world in (1, 2, 4, 8):
        comm = projection_comm(n, world, dev)
        g, f = comm.rows_of(st.estimate), comm.rows_of(st.residual)
        ctr = P.MulCounter()
        NS.composite_step(comm, g, f, sp.matrix, sp.precond, sp.residual, sp.matrix,
                          (2, 3, 4, 5), 2, ctr)  # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            g2, f2 = NS.composite_step(comm, g, f, sp.matrix, sp.precond, sp.residual, sp.matrix,
                                       (2, 3, 4, 5), 2, ctr)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        base = base or ms
        out[f"P{world}"] = {"ms_per_step_rank0": ms, "compute_efficiency": base / (world * ms)}
        print(world, json.dumps(out[f"P{world}"]), flush=True)
        comm.close()
        del g, f, g2, f2
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open(f"gpurun_out/native_projection_{args.gemm}.json", "w"), indent=1)


if __name__ == "__main__":
    main()
