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
are combined by an ordered binary tree -- one reduction -- whose every combine
runs block-row sharded over the union of the two groups' ranks; the root of the
tree covers all ranks, which hold the state block-row sharded, compute
S_n(F) G together and assemble G', F' together.  Inside a group the products
are block-row sharded too (:class:`~paper_2008_11480_b200.sharded.ShardedEngine`
on a sub-communicator), so e.g. 8 GPUs and 4 parts run 4 groups of 2.

Same GEMM DAG size as the reference: every part product, 2 per fold/combine
(the tree performs k - 1 combines like the left fold), S_n and the two
assembly products -- 22 products per step for rates (2, 3, 4, 5), order_n = 2;
:meth:`GroupedComposite.products_executed` sums them over the groups.  With
one group the evaluation order is the reference's and the result is bitwise
the single-GPU ``composite_step``; with several, the tree's association
differs from the left fold, so agreement is within the FP64 tolerance
(rounding at the kappa(A) u level), not bitwise.

The exchange of a combine is point-to-point (``torch.distributed``
``batch_isend_irecv``: NCCL over NVLink on GPUs; gloo isend/irecv in the CPU
tests): the union's ranks receive their rows of the left range's (t, r) and the
right range's (t, r) in full.  Work is partitioned by a cost model (products
per part divided by the group size, combines divided by the union size) that
picks group sizes and the contiguous segmentation with the shortest critical
path.
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


def _tree_levels(ngroups: int):
    """Ordered binary tree over the groups: per level d = 1, 2, 4, ... the
    combines (lo, mid, hi) of group ranges L = [lo, mid), R = [mid, hi)."""
    out = []
    d = 1
    while d < ngroups:
        out.append([(i, i + d, min(i + 2 * d, ngroups)) for i in range(0, ngroups, 2 * d)
                    if i + d < ngroups])
        d *= 2
    return out


def _critical_path(segments, sizes, costs, order_n) -> float:
    """Time (in products of one GPU) until every rank has its rows of G', F':
    S_n(F) G block-row over all ranks, each group's parts and fold block-row
    over the group, every tree combine block-row over the union of its two
    ranges, G' and F' block-row over all ranks."""
    world = sum(sizes)
    pre = (order_n - 1) / world
    ready = [pre + (sum(costs[i] for i in seg) + 2 * (len(seg) - 1)) / sizes[gi]
             for gi, seg in enumerate(segments)]
    for level in _tree_levels(len(segments)):
        for lo, mid, hi in level:
            ready[lo] = max(ready[lo], ready[mid]) + 2 / sum(sizes[lo:hi])
    return ready[0] + 2 / world


def _compositions(total: int, parts: int):
    """Ordered ways to write ``total`` as ``parts`` positive integers."""
    for cuts in itertools.combinations(range(1, total), parts - 1):
        b = (0,) + cuts + (total,)
        yield [b[i + 1] - b[i] for i in range(parts)]


def plan_groups(world: int, costs, order_n: int):
    """Split ``world`` ranks into G = min(world, parts) contiguous groups and the
    parts into G contiguous segments, choosing group sizes and segmentation with
    the shortest critical path (ties: the first found, near-equal sizes first).
    Returns (groups, segments): lists of rank lists and of part-index lists."""
    k = len(costs)
    if k < 1:
        raise ValueError("composite spec needs at least one rate")
    g = max(1, min(world, k))
    even = [r1 - r0 for r0, r1 in row_splits(world, g)]
    size_opts = [even] + [s for s in _compositions(world, g) if s != even]
    best, best_t = None, None
    for sizes in size_opts:
        for cuts in itertools.combinations(range(1, k), g - 1):
            bounds = (0,) + cuts + (k,)
            segs = [list(range(bounds[i], bounds[i + 1])) for i in range(g)]
            t = _critical_path(segs, sizes, costs, order_n)
            if best_t is None or t < best_t - 1e-9:
                best, best_t = (sizes, segs), t
    sizes, segs = best
    groups, r = [], 0
    for sz in sizes:
        groups.append(list(range(r, r + sz)))
        r += sz
    return groups, segs


class GroupedComposite:
    """The composite step with its parts on GPU groups and one tree reduction.

    Every rank holds A, S^-1, B (replicated).  The state (G, F) and theta are
    block-row sharded over all ranks (``world_eng``), like the block-row path:
    S_n(F) G and the assembly G' = t + r S_n(F) G, F' = I - G' A use every GPU.
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
        self.levels = _tree_levels(len(self.groups))
        self.gid = next(i for i, g in enumerate(self.groups) if self.rank in g)
        self._stage = self.world > 1 and dist.get_backend() == "gloo"
        self.bytes_moved = 0

        def ranks_of(lo, hi):
            return [r for g in self.groups[lo:hi] for r in g]

        # communicators: every rank creates every subgroup, in the same order; a
        # range covering all ranks uses the default group
        ranges = [tuple(g) for g in self.groups]
        for level in self.levels:
            ranges += [tuple(ranks_of(lo, hi)) for lo, _, hi in level]
        pgs = {}
        for rr in ranges:
            if rr in pgs:
                continue
            if len(rr) == self.world:
                pgs[rr] = None
            else:
                pg = dist.new_group(list(rr)) if self.world > 1 else None
                pgs[rr] = pg
        engines = {}

        def engine(rr):
            rr = tuple(rr)
            if rr not in engines:
                comm = RowComm(n, group=pgs.get(rr)) if self.rank in rr else None
                engines[rr] = ShardedEngine(comm, ops=ops, prefetch=prefetch) if comm else None
            return engines[rr]

        self.world_eng = engine(tuple(range(self.world)))
        self.group_eng = engine(self.groups[self.gid])
        # this rank's combines: (L ranks, R ranks, union engine) per level
        self.plan = []
        for level in self.levels:
            for lo, mid, hi in level:
                u = ranks_of(lo, hi)
                if self.rank in u:
                    self.plan.append((ranks_of(lo, mid), ranks_of(mid, hi), engine(u)))
        self._engines = [e for e in engines.values() if e is not None]
        # the exchange of the tree uses point-to-point ops: wire them up front
        # (NCCL's batched p2p needs the pair communicators' first use collective)
        self.eng = self.world_eng
        self.comm = self.world_eng.comm

    # -- helpers ---------------------------------------------------------------
    @property
    def ctr(self) -> MulCounter:
        """This rank's products (each rank of a communicator ticks once per
        product of that communicator)."""
        c = MulCounter()
        for e in self._engines:
            c.mmm += e.ctr.mmm
            c.mvm += e.ctr.mvm
        return c

    def products_executed(self) -> int:
        """Products over all groups so far (each communicator's leader counts)."""
        own = sum(e.ctr.mmm for e in self._engines if e.comm.rank == 0)
        if self.world == 1:
            return own
        dev = "cuda" if self.dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([float(own)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t)
        return int(t.item())

    def _move(self, blocks, count: int, src, dst, full: bool, like: torch.Tensor):
        """Row blocks of ``count`` matrices held by the ranks ``src`` (near-equal
        row split over them; ``blocks`` on src ranks) -> on the ranks ``dst``
        either the full matrices (``full``) or their rows of dst's split.
        Point-to-point; returns a list on dst ranks, else None."""
        n = self.n
        me = self.rank
        ssplit = row_splits(n, len(src))
        dsplit = row_splits(n, len(dst))

        def want(t):
            return (0, n) if full else dsplit[dst.index(t)]

        ops, out, copies = [], None, []
        if me in dst:
            c, d = want(me)
            out = [torch.empty((d - c, n), dtype=torch.float64, device=like.device)
                   for _ in range(count)]
            for j in range(count):
                for si, s in enumerate(src):
                    a, b = ssplit[si]
                    lo, hi = max(a, c), min(b, d)
                    if lo >= hi:
                        continue
                    if s == me:
                        out[j][lo - c:hi - c].copy_(blocks[j][lo - a:hi - a])
                    elif self._stage:
                        buf = torch.empty((hi - lo, n), dtype=torch.float64)
                        ops.append(("recv", buf, s))
                        copies.append((out[j][lo - c:hi - c], buf))
                    else:
                        ops.append(("recv", out[j][lo - c:hi - c], s))
        if me in src:
            a, b = ssplit[src.index(me)]
            for j in range(len(blocks)):
                for t in dst:
                    if t == me:
                        continue
                    c, d = want(t)
                    lo, hi = max(a, c), min(b, d)
                    if lo >= hi:
                        continue
                    x = blocks[j][lo - a:hi - a].contiguous()
                    if self._stage:
                        x = x.cpu()
                    ops.append(("send", x, t))
                    self.bytes_moved += x.numel() * 8
        if ops:
            if self._stage:  # gloo: tagged, non-blocking point-to-point
                works = [self.dist.isend(x, p) if k == "send" else self.dist.irecv(x, p)
                         for k, x, p in ops]
            else:  # NCCL: one group, no ordering constraints between peers
                works = self.dist.batch_isend_irecv(
                    [self.dist.P2POp(self.dist.isend if k == "send" else self.dist.irecv, x, p)
                     for k, x, p in ops])
            for w in works:
                w.wait()
        for dstv, buf in copies:
            dstv.copy_(buf)
        return out

    def _segment(self, a: Sharded, precond: Sharded, residual: Sharded):
        """Left fold over this group's parts (newton_schulz.py:204-216)."""
        eng = self.group_eng
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
        return eng.rows_of(t_c), eng.rows_of(r_c)

    # -- the step ----------------------------------------------------------------
    def step(self, g: Sharded, f: Sharded, a: Sharded, precond: Sharded, residual: Sharded):
        """One composite step on world-split row blocks ``g``, ``f`` (Sharded of
        ``world_eng``); returns the (G', F') row blocks."""
        W = self.world_eng
        nsp = W.horner(f, g, self.order_n)  # state part, block-row over all ranks
        t, r = self._segment(a, precond, residual)
        like = W.rows_of(a)
        for left, right, ue in self.plan:
            # my current blocks belong to `left` or `right` (their owners' split)
            union = left + right
            t_l, r_l = self._move([t, r] if self.rank in left else [], 2, left, union, False, like)
            t_r, r_r = self._move([t, r] if self.rank in right else [], 2, right, union, True, like)
            t = ue.ops.gemm(r_l, t_r, 1.0, t_l, 1.0, 0.0, ue.comm.r0, False, ue.ctr)
            r = ue.ops.gemm(r_l, r_r, 1.0, None, 0.0, 0.0, ue.comm.r0, False, ue.ctr)
            del t_l, r_l, t_r, r_r
        if self.plan:
            assert self.plan[-1][2].comm.world == self.world
        g_new = W.mm(W.local(r), nsp, c=W.local(t), beta=1.0)
        f_new = W.residual(g_new, a, gather=False)  # F is only ever a left operand
        return g_new, f_new

    def plain_richardson(self, theta: Sharded, p: Sharded, a: Sharded, b: Sharded):
        """theta - P (A theta - b) with world-split P."""
        return self.world_eng.plain_richardson(theta, p, a, b)

