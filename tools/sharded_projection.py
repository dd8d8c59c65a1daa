"""Compute-only strong-scaling projection of the block-row sharded C4 step on
one GPU: rank 0's share of the step (its row block of every product, the
replicated operands, the exact DAG of sharded.py) timed for P = 1, 2, 4, 8
with the exchange replaced by an already-gathered operand.  Together with the
exchange volume per rank this bounds the multi-GPU step from below; it is a
projection, not a multi-GPU measurement.  Prints one JSON object."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import configs  # noqa: E402
from paper_2008_11480_b200.sharded import ShardedEngine, row_splits  # noqa: E402


class ProjComm:
    """Rank 0 of P ranks; gathers return a resident full-size operand (the
    exchange itself is not timed)."""

    def __init__(self, n, world):
        self.n, self.world, self.rank = n, world, 0
        self.splits = row_splits(n, world)
        self.r0, self.r1 = self.splits[0]
        self.bytes_gathered = 0
        self._full = {}

    def _buf(self, cols, dev):
        if cols not in self._full:
            self._full[cols] = torch.zeros((self.n, cols), dtype=torch.float64, device=dev)
        return self._full[cols]

    def start_gather(self, local):
        self.bytes_gathered += (self.n - local.shape[0]) * local.shape[1] * 8
        return (None, self._buf(local.shape[1], local.device))

    def finish(self, pending):
        return pending[1]

    def all_reduce_sum(self, x):
        return x


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    a, b = configs.c4_householder_device(n=n, rhs=64)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    del a
    st = P.initial_series(sp, 0, 1, order=2)
    out = {"n": n, "note": "rank 0's products only; exchange replaced by a resident operand"}
    for world in (1, 2, 4, 8):
        comm = ProjComm(n, world)
        eng = ShardedEngine(comm, prefetch=False)
        A, Pm, B = eng.replicated(sp.matrix), eng.replicated(sp.precond), eng.replicated(sp.residual)
        g = eng.local(st.estimate[comm.r0:comm.r1].clone())
        f = eng.local(st.residual[comm.r0:comm.r1].clone())
        th, bb = eng.replicated(torch.zeros_like(b)), eng.replicated(b)
        eng.composite_step(g, f, A, Pm, B, (2, 3, 4, 5), 2)  # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 2
        for _ in range(reps):
            th2 = eng.plain_richardson(th, g, A, bb)
            g2, f2 = eng.composite_step(g, f, A, Pm, B, (2, 3, 4, 5), 2)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3 / reps
        out[f"P{world}"] = {"rows": comm.r1 - comm.r0, "rank0_step_s": sec,
                            "exchange_bytes_per_rank": comm.bytes_gathered // (reps + 1)}
        del eng, g, f, g2, f2, th2, comm
        torch.cuda.empty_cache()
    t1 = out["P1"]["rank0_step_s"]
    for world in (2, 4, 8):
        d = out[f"P{world}"]
        d["compute_scaling_efficiency"] = t1 / (world * d["rank0_step_s"])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
