"""Compute-only strong-scaling projection of the block-row sharded C5 step
(recursive Richardson / factorised order 16, 18 products + 2 n^2 r, n=32768,
256 RHS) on one GPU: rank 0's share of a steady-state step (its row block of
every product, replicated A / b / theta, the DAG of sharded.py) timed for
P = 1, 2, 4, 8, with the exchange replaced by an already-gathered operand.
Together with the exchange volume per rank this bounds the multi-GPU step from
below; it is a projection, not a multi-GPU measurement.  Prints one JSON object.

    python tools/sharded_projection_c5.py [n]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import configs  # noqa: E402
from paper_2008_11480_b200.sharded import ShardedEngine  # noqa: E402

from sharded_projection import ProjComm  # noqa: E402  (rank 0 of P, resident gathers)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a, b = configs.c5_gram_device(n=n, m=int(n * 40000 / 32768), rhs=256)
sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
del a
st = P.initial_richardson(sp, b, 0, 1, order=16, q=16)
A_full = sp.matrix
del sp
torch.cuda.empty_cache()
plan16 = P.plan_order(16)
out = {"n": n, "rhs": 256,
       "dag": "richardson_recursive_step, factorised order 16 (18 n^3 products) + 2 n^2 r",
       "note": "rank 0's products only; exchange replaced by a resident operand"}
for world in (8, 4, 2, 1):  # P = 1 last: it releases the initial state to fit one GPU
    comm = ProjComm(n, world)
    eng = ShardedEngine(comm, prefetch=False)
    rows = slice(comm.r0, comm.r1)
    inner = st.inner
    take = (lambda m: m[rows]) if world == 1 else (lambda m: m[rows].clone())
    state = [eng.local(take(m)) for m in (inner.estimate, inner.residual, inner.accel_estimate,
                                          inner.accel_residual)]
    A, bb, th = eng.replicated(A_full), eng.replicated(b), eng.replicated(st.theta)
    del inner
    if world == 1:
        st = None
    # first call builds the carried omega / N (untimed), then one steady-state step
    g, f, l, r, om, ns, th = eng.richardson_recursive_step(*state, None, None, A, th, bb, 16,
                                                           factor_plan=plan16, doubling_sum=True)
    del state
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    c0, b0 = eng.ctr.mmm, comm.bytes_gathered
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = eng.richardson_recursive_step(g, f, l, r, om, ns, A, th, bb, 16, factor_plan=plan16,
                                        doubling_sum=True)
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    out[f"P{world}"] = {"rows": comm.r1 - comm.r0, "rank0_step_s": sec,
                        "products": eng.ctr.mmm - c0,
                        "exchange_bytes_per_rank_per_step": comm.bytes_gathered - b0}
    del eng, g, f, l, r, om, ns, res, comm
    torch.cuda.empty_cache()
t1 = out["P1"]["rank0_step_s"]
for world in (2, 4, 8):
    d = out[f"P{world}"]
    d["compute_scaling_efficiency"] = t1 / (world * d["rank0_step_s"])
print(json.dumps(out, indent=1))
