"""Compute-only projection of the grouped composite step (grouped.py: composite
parts on GPU groups + one ordered tree reduction) on one GPU.

For P = 2, 4, 8 the cost model's plan (group sizes, part segments) is taken
from grouped.plan_groups; every piece of the critical path is then timed as
one rank's share of it on this GPU -- S_n(F) G on n/P rows, each group's parts
and fold on n/size rows (right operands replicated, as after a gather), each
tree combine on n/union rows, the assembly on n/P rows -- and combined with the
same critical-path rule as the planner.  Exchange times are not included
(they are reported as bytes per rank).  A projection, not a multi-GPU
measurement.  Prints one JSON object: python tools/grouped_projection.py [n]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import configs  # noqa: E402
from paper_2008_11480_b200.grouped import _tree_levels, part_cost, plan_groups  # noqa: E402
from paper_2008_11480_b200.sharded import Sharded, ShardedEngine, row_splits  # noqa: E402

RATES = (2, 3, 4, 5)


class Rows:
    """One rank's row block of a ``world``-way split; gathers are not timed."""

    def __init__(self, n, world):
        self.n, self.world, self.rank = n, world, 0
        self.splits = row_splits(n, world)
        self.r0, self.r1 = self.splits[0]
        self._full = {}

    def start_gather(self, local):
        key = local.shape[1]
        if key not in self._full:
            self._full[key] = torch.zeros((self.n, key), dtype=torch.float64, device=local.device)
        return (None, self._full[key])

    def finish(self, pending):
        return pending[1]


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a, _ = configs.c4_householder_device(n=n, rhs=1)
sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
del a
st = P.initial_series(sp, 0, 1, order=2)
costs = [part_cost(x) for x in RATES]


def engine(world):
    return ShardedEngine(Rows(n, world), prefetch=False)


def seg_time(seg, size):
    eng = engine(size)
    A, Pm, B = (eng.replicated(x) for x in (sp.matrix, sp.precond, sp.residual))

    def run():
        t_c = r_c = None
        for i in seg:
            t = eng.geometric(B, Pm, RATES[i], A)
            g = eng.residual(t, A)
            if t_c is None:
                t_c, r_c = t, g
            else:
                t_c = eng.mm(r_c, t, c=t_c, beta=1.0)
                r_c = eng.mm(r_c, g)
    return timed(run)


def two_products(world):
    """A combine / the assembly: two products on n/world rows."""
    eng = engine(world)
    rows = eng.comm.r1 - eng.comm.r0
    x = eng.local(st.residual[:rows].clone())
    y = eng.replicated(st.estimate)

    def run():
        eng.mm(x, y, c=x, beta=1.0)
        eng.mm(x, y)
    return timed(run)


def ns_time(world):
    eng = engine(world)
    rows = eng.comm.r1 - eng.comm.r0
    f = eng.local(st.residual[:rows].clone())
    g = eng.local(st.estimate[:rows].clone())
    return timed(lambda: eng.horner(f, g, 2))


full = {"P1_step_s": None}
eng1 = engine(1)
A1, P1, B1 = (eng1.replicated(x) for x in (sp.matrix, sp.precond, sp.residual))
full["P1_step_s"] = timed(lambda: eng1.composite_step(eng1.local(st.estimate),
                                                      eng1.local(st.residual), A1, P1, B1,
                                                      RATES, 2))
out = {"n": n, "rates": RATES, "note": "compute only; one rank's share of each piece",
       "P1_step_s": full["P1_step_s"]}
for world in (2, 4, 8):
    groups, segs = plan_groups(world, costs, 2)
    sizes = [len(g) for g in groups]
    pre = ns_time(world)
    ready = [pre + seg_time(seg, sz) for seg, sz in zip(segs, sizes)]
    moved = 0
    for level in _tree_levels(len(groups)):
        for lo, mid, hi in level:
            u = sum(sizes[lo:hi])
            ready[lo] = max(ready[lo], ready[mid]) + two_products(u)
            moved = max(moved, (2 * n * n + 2 * n * n // u) * 8)  # full right (t, r) + own left rows
    step = ready[0] + two_products(world)
    out[f"P{world}"] = {"group_sizes": sizes, "segments": segs, "critical_path_s": step,
                        "compute_efficiency": full["P1_step_s"] / (world * step),
                        "max_bytes_received_per_rank_per_combine": moved}
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
