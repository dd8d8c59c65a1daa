"""Composite expansion with its independently-rated parts on GPU groups.

``composite_step`` (newton_schulz.py:177-228) evaluates, per rate x_i, the part
T_i = sum_{j<x_i} B^j S^-1 and Gamma_i = I - T_i A (ns:204-210), folds them
left to right (ns:212-216)

    t <- t + r T_i,   r <- r Gamma_i

and assembles G' = t + r S_n(F) G, F' = I - G' A (ns:218-220).  The parts
depend only on the splitting, not on the state, so they can run on different
GPUs at the same time.  The fold is associative as an operation on pairs,

    (t1, r1) (+) (t2, r2) = (t1 + r1 t2, r1 r2),

so each GPU group folds a contiguous segment of the parts locally (left to
right, exactly the reference's fold inside the segment) and the segment results
are combined by an ordered binary tree -- one reduction -- into the root group,
which holds the state, computes S_n(F) G while the other groups work on their
parts, and assembles G', F'.  Inside a group the products are block-row
sharded (:class:`~paper_2008_11480_b200.sharded.ShardedEngine` on a
sub-communicator), so e.g. 8 GPUs and 4 parts run 4 groups of 2.

Same GEMM DAG size as the reference: every part product, 2 per fold/combine
(the tree performs k - 1 combines like the left fold), S_n and the two
assembly products -- 22 products per step for rates (2, 3, 4, 5), order_n = 2;
:meth:`GroupedComposite.products_executed` sums them over the groups.  With
one group the evaluation order is the reference's and the result is bitwise
the single-GPU ``composite_step``; with several, the tree's association
differs from the left fold, so agreement is within the FP64 tolerance
(rounding at the kappa(A) u level), not bitwise.

The pair exchange of the tree is point-to-point (``torch.distributed``
isend/irecv: NCCL over NVLink on GPUs, gloo in the CPU tests): every rank of
the sending group ships its row blocks of (t, r) to every rank of the
receiving group.  Work is partitioned by a cost model (products per part,
divided by the group size) that picks the contiguous segmentation with the
shortest critical path.
"""

from __future__ import annotations

import itertools

import torch

from .matrix_core import MulCounter
from .sharded import RowComm, Sharded, ShardedEngine, row_splits

__all__ = ["GroupedComposite", "part_cost", "plan_groups"]


class _SoloComm:
    """One-rank comm for dry runs (no process group)."""

    def __init__(self, n: int):
        self.world, self.rank = 1, 0
        self.splits = [(0, n)]
        self.r0, self.r1 = 0, n

    def start_gather(self, local):
        return (None, local)

    def finish(self, pending):
        return pending[1]


class _CountOps:
    """Dry-run local ops: counts products, computes nothing of interest."""

    def gemm(self, a, b, alpha, c, beta, diag, doff, is_mv, ctr, out=None):
        if is_mv:
            ctr.mvm += 1
        else:
            ctr.mmm += 1
        return torch.zeros((a.shape[0], b.shape[1]), dtype=torch.float64)

    def lin(self, cdiag, doff, terms, rows, cols, like):
        return torch.zeros((rows, cols), dtype=torch.float64)

    def sumsq(self, x):
        return 0.0


def part_cost(x: int) -> int:
    """Products of one composite part of rate x: T_x (series_toolkit.py:432-457)
    plus its residual Gamma = I - T A (newton_schulz.py:209-210)."""
    eng = ShardedEngine(_SoloComm(2), ops=_CountOps())
    z = eng.replicated(torch.zeros((2, 2), dtype=torch.float64))
    t = z if x == 1 else eng.geometric(z, z, x, z)
    eng.residual(t, z)
    return eng.ctr.mmm


def _critical_path(segments, sizes, costs, order_n) -> float:
    """Time (in products of one GPU) until the root group has G', F'."""
    ready = []
    for gi, seg in enumerate(segments):
        work = sum(costs[i] for i in seg) + 2 * (len(seg) - 1)
        if gi == 0:
            work += order_n - 1  # S_n(F) G on the root group
        ready.append(work / sizes[gi])
    g = len(segments)
    d = 1
    while d < g:
        for i in range(0, g, 2 * d):
            if i + d < g:
                ready[i] = max(ready[i], ready[i + d]) + 2 / sizes[i]
        d *= 2
    return ready[0] + 2 / sizes[0]


def plan_groups(world: int, costs, order_n: int):
    """Split ``world`` ranks into G = min(world, parts) contiguous groups of
    near-equal size and the parts into G contiguous segments, choosing the
    segmentation with the shortest critical path.  Returns (groups, segments):
    lists of rank lists and of part-index lists."""
    k = len(costs)
    if k < 1:
        raise ValueError("composite spec needs at least one rate")
    g = max(1, min(world, k))
    groups = [list(range(r0, r1)) for r0, r1 in row_splits(world, g)]
    sizes = [len(x) for x in groups]
    best, best_t = None, None
    for cuts in itertools.combinations(range(1, k), g - 1):
        bounds = (0,) + cuts + (k,)
        segs = [list(range(bounds[i], bounds[i + 1])) for i in range(g)]
        t = _critical_path(segs, sizes, costs, order_n)
        if best_t is None or t < best_t - 1e-12:
            best, best_t = segs, t
    return groups, best


class GroupedComposite:
    """The composite step with its parts on GPU groups and one tree reduction.

    Every rank holds A, S^-1, B (replicated); the state (G, F) and theta live
    on the root group (group 0) as row blocks of its sub-communicator.
    ``ops`` injects the local-ops layer (CPU in the gloo tests); the default is
    the DMMA library."""

    def __init__(self, n: int, rates, order_n: int = 2, ops=None, prefetch: bool = True):
        import torch.distributed as dist

        if order_n < 1:
            raise ValueError("order_n must be >= 1")
        self.n = n
        self.rates = tuple(int(x) for x in rates)
        if any(x < 1 for x in self.rates):
            raise ValueError("rates must be >= 1")
        self.order_n = order_n
        self.dist = dist
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.costs = [part_cost(x) for x in self.rates]
        self.groups, self.segments = plan_groups(self.world, self.costs, order_n)
        self.gid = next(i for i, g in enumerate(self.groups) if self.rank in g)
        pg = None
        if self.world > 1:
            # every rank creates every subgroup, in the same order
            for i, ranks in enumerate(self.groups):
                h = dist.new_group(ranks)
                if i == self.gid:
                    pg = h
        self.comm = RowComm(n, group=pg)
        self.eng = ShardedEngine(self.comm, ops=ops, prefetch=prefetch)
        self.is_root = self.gid == 0
        self.bytes_sent = 0
        # gloo point-to-point moves host memory only: stage device blocks through
        # the host (the 1-GPU test mode that runs every rank on cuda:0)
        self._stage = self.world > 1 and dist.get_backend() == "gloo"

    # -- helpers ---------------------------------------------------------------
    @property
    def ctr(self) -> MulCounter:
        """This rank's counter (each rank of a group ticks once per group product)."""
        return self.eng.ctr

    def products_executed(self) -> int:
        """Products over all groups so far (group leaders' counters summed)."""
        own = self.eng.ctr.mmm if self.comm.rank == 0 else 0
        if self.world == 1:
            return own
        dev = "cuda" if self.dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([float(own)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t)
        return int(t.item())

    def _send_pair(self, t: Sharded, r: Sharded, dst_group: int):
        """Ship this rank's row blocks of (t, r) to every rank of ``dst_group``."""
        works = []
        for v in (t, r):
            blk = self.eng.rows_of(v).contiguous()
            if self._stage and blk.is_cuda:
                blk = blk.cpu()
            for dst in self.groups[dst_group]:
                works.append(self.dist.isend(blk, dst))
                self.bytes_sent += blk.numel() * blk.element_size()
        for w in works:
            w.wait()

    def _recv_pair(self, src_group: int, like: torch.Tensor):
        """Full (t, r) of ``src_group``, assembled from its ranks' row blocks."""
        src = self.groups[src_group]
        splits = row_splits(self.n, len(src))
        dev = "cpu" if self._stage else like.device
        fulls, works = [], []
        for _ in range(2):
            full = torch.empty((self.n, self.n), dtype=torch.float64, device=dev)
            for s, (r0, r1) in zip(src, splits):
                works.append(self.dist.irecv(full[r0:r1], s))
            fulls.append(full)
        for w in works:
            w.wait()
        if self._stage and like.is_cuda:
            fulls = [x.to(like.device) for x in fulls]
        return fulls

    def _segment(self, a: Sharded, precond: Sharded, residual: Sharded):
        """Left fold over this group's parts (newton_schulz.py:204-216)."""
        eng = self.eng
        t_c = r_c = None
        for i in self.segments[self.gid]:
            x = self.rates[i]
            t = Sharded(eng.rows_of(precond).clone(), False) if x == 1 else \
                eng.geometric(residual, precond, x, a)
            gam = eng.residual(t, a)
            if t_c is None:
                t_c, r_c = t, gam
            else:
                t_c = eng.mm(r_c, t, c=t_c, beta=1.0)
                r_c = eng.mm(r_c, gam)
        return t_c, r_c

    # -- the step ----------------------------------------------------------------
    def step(self, g: Sharded | None, f: Sharded | None, a: Sharded, precond: Sharded,
             residual: Sharded):
        """One composite step.  On root-group ranks ``g``/``f`` are this rank's row
        blocks and (G', F') row blocks are returned; elsewhere they are ignored
        and (None, None) is returned."""
        eng = self.eng
        nsp = None
        if self.is_root:
            if g is None or f is None:
                raise ValueError("the root group needs the state (g, f)")
            nsp = eng.horner(f, g, self.order_n)  # state part, overlaps the others' parts
        t_c, r_c = self._segment(a, precond, residual)
        ng = len(self.groups)
        d = 1
        while d < ng:
            if self.gid % (2 * d) == d:
                self._send_pair(t_c, r_c, self.gid - d)
                return None, None
            if self.gid % (2 * d) == 0 and self.gid + d < ng:
                t_r, r_r = self._recv_pair(self.gid + d, eng.rows_of(a))
                t_c = eng.mm(r_c, eng.replicated(t_r), c=t_c, beta=1.0)
                r_c = eng.mm(r_c, eng.replicated(r_r))
                del t_r, r_r
            d *= 2
        g_new = eng.mm(r_c, nsp, c=t_c, beta=1.0)
        f_new = eng.residual(g_new, a, gather=False)  # F is only ever a left operand
        return g_new, f_new

    def plain_richardson(self, theta: Sharded, p: Sharded, a: Sharded, b: Sharded):
        """theta - P (A theta - b) on the root group."""
        if not self.is_root:
            return theta
        return self.eng.plain_richardson(theta, p, a, b)
