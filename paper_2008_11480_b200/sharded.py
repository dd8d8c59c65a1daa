"""Block-row sharded hot path over several GPUs.

Every state matrix is split into contiguous row blocks, one per rank; A and
the splitting (S^-1, B) are replicated.  A product ``L @ R`` produces the
local rows ``L[rows] @ R`` -- no communication when R is replicated (every
``I - X A`` residual and every product with B or S^-1), one all-gather of R's
row panels when R is itself sharded.  The local products run on the library's
DMMA kernels through ``si_gemm_ex`` with the ``diag * I`` term shifted to the
block's global diagonal; the K accumulation order is the single-GPU one, so
results are independent of the number of ranks.

The GEMM DAG is the reference's (series_toolkit.py:263-457,
newton_schulz.py:177-228, richardson.py:81-189), so ``MulCounter`` deltas
match the single-GPU path and the reference tick for tick.  The row-panel
exchange is pluggable: :class:`~paper_2008_11480_b200.peer.PeerComm` (copy
engines over CUDA IPC, products gated per panel inside the DMMA kernel -- the
product path) or :class:`RowComm` (``torch.distributed`` all-gather: NCCL as
the baseline, gloo in the CPU tests).  The local-ops layer is injectable so
the orchestration can be exercised on CPU, but the product default
(:class:`CudaOps`) has no host path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .matrix_core import MulCounter
from .series_toolkit import FactorPlan, Horner, Lin, Mul, PrimeWrap, Residual, Split, TableForm
from .series_toolkit import geometric_base_plan

__all__ = ["CudaOps", "RowComm", "Sharded", "ShardedEngine", "row_splits"]


def row_splits(n: int, world: int) -> list[tuple[int, int]]:
    """Near-equal contiguous row blocks [(r0, r1), ...]."""
    base, extra = divmod(n, world)
    out, r = [], 0
    for p in range(world):
        rows = base + (1 if p < extra else 0)
        out.append((r, r + rows))
        r += rows
    return out


class RowComm:
    """All-gather of row blocks over a torch.distributed process group."""

    def __init__(self, n: int, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.splits = row_splits(n, self.world)
        self.r0, self.r1 = self.splits[self.rank]
        self.pad = max(r1 - r0 for r0, r1 in self.splits)
        self.bytes_gathered = 0

    def all_gather_rows(self, local: torch.Tensor) -> torch.Tensor:
        return self.finish(self.start_gather(local))

    def start_gather(self, local: torch.Tensor):
        """Launch the all-gather of a row block (asynchronous on NCCL's stream);
        ``finish`` makes the caller's stream wait and returns the full matrix."""
        if self.world == 1:
            return (None, local)
        cols = local.shape[1]
        rows = local.shape[0]
        if rows < self.pad:
            padded = torch.zeros((self.pad, cols), dtype=local.dtype, device=local.device)
            padded[:rows] = local
        else:
            padded = local.contiguous()
        out = torch.empty((self.world * self.pad, cols), dtype=local.dtype, device=local.device)
        work = self.dist.all_gather_into_tensor(out, padded, group=self.group, async_op=True)
        self.bytes_gathered += out.numel() * out.element_size()
        return (work, out)

    def finish(self, pending) -> torch.Tensor:
        work, out = pending
        if work is None:
            return out
        work.wait()
        if all(r1 - r0 == self.pad for r0, r1 in self.splits):
            return out
        return torch.cat([out[p * self.pad:p * self.pad + (r1 - r0)]
                          for p, (r0, r1) in enumerate(self.splits)])

    def barrier(self):
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def all_reduce_sum(self, x: float) -> float:
        """Scalar sum over the ranks (the one reduction of the stop rule)."""
        if self.world == 1:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())


class CudaOps:
    """Local products and sums on the DMMA library (no host fallback)."""

    def gemm(self, a, b, alpha, c, beta, diag, doff, is_mv, ctr: MulCounter, out=None):
        m, k = a.shape
        n = b.shape[1]
        a = a.contiguous()
        if c is not None:
            c = c.contiguous()
        if out is None:
            out = torch.empty((m, n), dtype=torch.float64, device=a.device)
        buf = _lib.counter_buf()
        if not isinstance(b, torch.Tensor):  # peer.GatedOperand: panel-gated product
            _lib.call("si_gemm_panels", _lib.handle(a.device.index), m, n, k, alpha, a.data_ptr(),
                      k, b.t.data_ptr(), n, beta if c is not None else 0.0,
                      c.data_ptr() if c is not None else None, n, diag, doff, out.data_ptr(), n,
                      b.ready, b.epoch, _lib.i64_array(b.bounds), len(b.bounds) - 1, int(is_mv),
                      buf, _lib.stream_ptr(a.device))
            ctr.absorb(buf)
            return out
        b = b.contiguous()
        _lib.call("si_gemm_ex", _lib.handle(a.device.index), m, n, k, alpha, a.data_ptr(), k,
                  b.data_ptr(), n, beta if c is not None else 0.0,
                  c.data_ptr() if c is not None else None, n, diag, doff, out.data_ptr(), n,
                  int(is_mv), buf, _lib.stream_ptr(a.device))
        ctr.absorb(buf)
        return out

    def sumsq(self, x) -> float:
        """Sum of squares of a local block (si_fro_norm, squared)."""
        x2 = x.contiguous()
        out = ctypes.c_double()
        _lib.call("si_fro_norm", _lib.handle(x2.device.index), x2.shape[0], x2.shape[1],
                  x2.data_ptr(), x2.shape[1], ctypes.byref(out), _lib.stream_ptr(x2.device))
        return float(out.value) ** 2

    def lin(self, cdiag, doff, terms, rows, cols, like):
        out = torch.empty((rows, cols), dtype=torch.float64, device=like.device)
        xs = [t.contiguous() for _, t in terms]
        ptrs = (ctypes.c_void_p * max(len(xs), 1))(*[x.data_ptr() for x in xs])
        _lib.call("si_lincomb_ex", _lib.handle(like.device.index), rows, cols, cdiag, doff, len(xs),
                  _lib.f64_array([c for c, _ in terms]), ptrs,
                  _lib.i64_array([x.shape[1] for x in xs]), out.data_ptr(), cols,
                  _lib.stream_ptr(like.device))
        return out


@dataclass
class Sharded:
    """A matrix value: replicated (``full``) or this rank's row block (``rows``)."""

    t: torch.Tensor
    full: bool
    _gathered: torch.Tensor | None = None
    _pending: object | None = None
    _gated: object | None = None


class ShardedEngine:
    """Evaluators and steps on block-row sharded values.

    With ``prefetch`` (default) every product result that may serve as a right
    operand starts its all-gather as soon as it is produced, on NCCL's stream,
    so the transfer overlaps the products that follow; the first consumer waits
    on it.  Residuals ``I - X A`` are only ever left operands and are not
    gathered."""

    def __init__(self, comm: RowComm, ops=None, ctr: MulCounter | None = None,
                 prefetch: bool = True):
        self.comm = comm
        self.ops = ops if ops is not None else CudaOps()
        self.ctr = ctr if ctr is not None else MulCounter()
        self.prefetch = prefetch

    # -- value helpers ------------------------------------------------------
    def rows_of(self, v: Sharded) -> torch.Tensor:
        return v.t[self.comm.r0:self.comm.r1] if v.full else v.t

    def full_of(self, v: Sharded) -> torch.Tensor:
        if v.full:
            return v.t
        if v._gathered is None:
            pending = v._pending if v._pending is not None else self.comm.start_gather(v.t)
            v._gathered = self.comm.finish(pending)
        return v._gathered

    def operand_of(self, v: Sharded):
        """Right operand of a product: the full matrix, or -- with a peer-memory
        comm in fused mode -- a gated operand whose panels may still be in
        flight (the product waits for each panel inside the kernel)."""
        if v.full:
            return v.t
        if v._gathered is not None:
            return v._gathered
        if v._gated is not None:
            return v._gated
        gate = getattr(self.comm, "gate", None)
        if gate is not None and self.comm.world > 1:
            if v._pending is None:
                v._pending = self.comm.start_gather(v.t)
            g = gate(v._pending)
            if not isinstance(g, torch.Tensor):
                v._gated = g
                return g
            v._gathered = g
            return g
        return self.full_of(v)

    def _produced(self, t: torch.Tensor, gather: bool) -> Sharded:
        v = Sharded(t, False)
        if gather and self.prefetch and self.comm.world > 1:
            v._pending = self.comm.start_gather(t)
        return v

    def replicated(self, t: torch.Tensor) -> Sharded:
        return Sharded(t, True)

    def local(self, t: torch.Tensor) -> Sharded:
        return Sharded(t, False)

    def mm(self, lhs: Sharded, rhs: Sharded, alpha=1.0, c: Sharded | None = None, beta=0.0,
           diag=0.0, mv=False, gather: bool = True) -> Sharded:
        gather = gather and not mv
        r = self.operand_of(rhs)
        kw = {}
        out_rows = getattr(self.comm, "output_rows", None)
        if gather and self.prefetch and self.comm.world > 1 and out_rows is not None:
            kw["out"] = out_rows(r.shape[1])  # written in place into its exchange slot
        out = self.ops.gemm(self.rows_of(lhs), r, alpha,
                            self.rows_of(c) if c is not None else None, beta, diag, self.comm.r0,
                            mv, self.ctr, **kw)
        return self._produced(out, gather)

    def residual(self, x: Sharded, a: Sharded, gather: bool = True) -> Sharded:
        return self.mm(x, a, alpha=-1.0, diag=1.0, gather=gather)

    def lin(self, cdiag: float, terms, like: Sharded) -> Sharded:
        rows = self.comm.r1 - self.comm.r0
        loc = [(coef, self.rows_of(v)) for coef, v in terms]
        cols = self.rows_of(like).shape[1]
        return Sharded(self.ops.lin(cdiag, self.comm.r0, loc, rows, cols, self.rows_of(like)), False)

    # -- stop rule (newton_schulz.py:328-331, matrix_core.py:167-168) ----------
    def fro_norm(self, v: Sharded) -> float:
        """||V||_F of a row-sharded (or replicated) matrix: local sums of squares
        and one scalar all-reduce."""
        if v.full:
            return self.ops.sumsq(v.t) ** 0.5
        return self.comm.all_reduce_sum(self.ops.sumsq(v.t)) ** 0.5

    def converged(self, f: Sharded, n: int) -> bool:
        return self.fro_norm(f) <= 1e-13 * n ** 0.5

    # -- evaluators (series_toolkit.py:263-457) -----------------------------
    def horner(self, y: Sharded, x: Sharded, h: int) -> Sharded:
        z = x
        for _ in range(h - 1):
            z = self.mm(y, z, c=x, beta=1.0)
        return z

    def eval_node(self, node, y: Sharded, x: Sharded, a: Sharded) -> Sharded:
        if isinstance(node, FactorPlan):
            node = node.root
        if isinstance(node, Horner):
            return self.horner(y, x, node.order)
        if isinstance(node, Split):
            u = x if node.p == 0 else self.eval_node(node.inner, y, x, a)
            if node.w == 1:
                return u
            q = y if node.p == 0 else self.residual(u, a)
            return self.eval_node(node.outer, q, u, a)
        if isinstance(node, PrimeWrap):
            z = self.eval_node(node.inner, y, x, a)
            return self.mm(y, z, c=x, beta=1.0)
        if isinstance(node, TableForm):
            return self._program(node, y, x, a)
        raise TypeError(f"not a plan node: {node!r}")

    def _program(self, form: TableForm, y, x, a):
        env = {"Y": y, "X": x}
        res = x
        prog = form.program
        i = 0
        while i < len(prog):
            ins = prog[i]
            if isinstance(ins, Mul):
                nxt = prog[i + 1] if i + 1 < len(prog) else None
                fused = False
                if (isinstance(nxt, Lin) and nxt.const == 0.0 and len(nxt.terms) == 2
                        and all(cf == 1.0 for cf, _ in nxt.terms)
                        and ins.dst in (nxt.terms[0][1], nxt.terms[1][1])
                        and nxt.terms[0][1] != nxt.terms[1][1]
                        and not any(_reads(p, ins.dst) for p in prog[i + 2:])):
                    other = nxt.terms[0][1] if nxt.terms[1][1] == ins.dst else nxt.terms[1][1]
                    env[nxt.dst] = self.mm(env[ins.lhs], env[ins.rhs], c=env[other], beta=1.0)
                    res = env[nxt.dst]
                    i += 2
                    fused = True
                if not fused:
                    env[ins.dst] = self.mm(env[ins.lhs], env[ins.rhs])
                    res = env[ins.dst]
                    i += 1
                continue
            if isinstance(ins, Residual):
                env[ins.dst] = self.residual(env[ins.src], a)
            else:
                env[ins.dst] = self.lin(ins.const, [(cf, env[r]) for cf, r in ins.terms], x)
            res = env[ins.dst]
            i += 1
        return res

    def mat_pow_counted(self, y: Sharded, e: int) -> Sharded:
        base, result = y, None
        while e > 0:
            if e & 1:
                result = base if result is None else self.mm(result, base)
            e >>= 1
            if e:
                base = self.mm(base, base)
        return result

    def geometric(self, y: Sharded, x: Sharded, order: int, a: Sharded) -> Sharded:
        if order == 1:
            return Sharded(self.rows_of(x).clone(), False)
        if order <= 64:
            return self.eval_node(geometric_base_plan(order), y, x, a)
        half = order // 2
        t = self.geometric(y, x, half, a)
        yh = self.mat_pow_counted(y, half)
        z = self.mm(yh, t, c=t, beta=1.0)
        if order % 2:
            z = self.mm(y, z, c=x, beta=1.0)
        return z

    # -- steps ---------------------------------------------------------------
    def composite_step(self, g: Sharded, f: Sharded, a: Sharded, precond: Sharded,
                       residual: Sharded, rates, order_n: int):
        """newton_schulz.py:177-228 on row blocks; returns (G', F') row blocks."""
        if order_n < 1:
            raise ValueError("order_n must be >= 1")
        ts, gs = [], []
        for x in rates:
            t = Sharded(self.rows_of(precond).clone(), False) if x == 1 else \
                self.geometric(residual, precond, x, a)
            ts.append(t)
            gs.append(self.residual(t, a))
        t_c, r_c = ts[0], gs[0]
        for i in range(1, len(ts)):
            t_c = self.mm(r_c, ts[i], c=t_c, beta=1.0)
            r_c = self.mm(r_c, gs[i])
        nsp = self.horner(f, g, order_n)
        g_new = self.mm(r_c, nsp, c=t_c, beta=1.0)
        f_new = self.residual(g_new, a, gather=False)  # F is only ever a left operand
        return g_new, f_new

    def ns_step(self, g: Sharded, f: Sharded, a: Sharded, order: int, plan=None):
        """newton_schulz.py:150-174 on row blocks."""
        new = self.horner(f, g, order) if plan is None else self.eval_node(plan, f, g, a)
        return new, self.residual(new, a, gather=False)

    def identity_rows(self, like: Sharded) -> Sharded:
        rows = self.comm.r1 - self.comm.r0
        ref = self.rows_of(like)
        return Sharded(self.ops.lin(1.0, self.comm.r0, [], rows, ref.shape[1], ref), False)

    def power_sum(self, gamma: Sharded, n: int) -> Sharded:
        """richardson.py:101-108 on row blocks: I + gamma + ... + gamma^(n-1)."""
        acc = self.identity_rows(gamma)
        cur = None
        for _ in range(n - 1):
            cur = gamma if cur is None else self.mm(cur, gamma, gather=False)
            acc = self.lin(0.0, [(1.0, acc), (1.0, cur)], gamma)
        return acc

    def power_sum_doubling(self, gamma: Sharded, n: int) -> Sharded:
        """Opt-in S_2t = S_t + gamma^t S_t (n = 2^m), as si_richardson_recursive_step."""
        if n < 2 or n & (n - 1):
            raise ValueError("doubling power sum needs n = 2^m >= 2")
        s = self.lin(0.0, [(1.0, self.identity_rows(gamma)), (1.0, gamma)], gamma)
        pw = gamma
        t = 2
        while t < n:
            pw = self.mm(pw, pw)
            s = self.mm(pw, s, c=s, beta=1.0)
            t *= 2
        return s

    def richardson_recursive_step(self, g: Sharded, f: Sharded, l: Sharded, r: Sharded,
                                  omega: Sharded | None, ns_part: Sharded | None, a: Sharded,
                                  theta: Sharded, b: Sharded, order: int, factor_plan=None,
                                  doubling_sum: bool = False):
        """richardson.py:111-189 on row blocks (q == n).  Returns
        (G', F', L', R', omega', ns', theta') with theta' replicated."""
        vec = theta.t.ndim == 1
        if vec:
            theta = Sharded(theta.t.reshape(-1, 1), theta.full)
            b = Sharded(b.t.reshape(-1, 1), b.full)
        n = order
        if omega is None or ns_part is None:
            ns_prev = self.horner(f, g, n)
            om_prev = self.mm(r, ns_prev, c=l, beta=1.0)
        else:
            ns_prev, om_prev = ns_part, omega
        s = self.power_sum_doubling(r, n) if doubling_sum else self.power_sum(r, n)
        diff = self.lin(0.0, [(1.0, om_prev), (-1.0, ns_prev)], g)
        g_new = self.mm(s, diff, c=ns_prev, beta=1.0)
        f_new = self.residual(g_new, a, gather=False)
        ns_new = (self.eval_node(factor_plan, f_new, g_new, a) if factor_plan is not None
                  else self.horner(f_new, g_new, n))
        l_new = self.mm(s, l)
        r_new = self.residual(l_new, a)
        om_new = self.mm(r_new, ns_new, c=l_new, beta=1.0)
        resid = self.mm(a, theta, c=b, beta=-1.0, mv=True)
        th = self.mm(om_new, resid, alpha=-1.0, c=theta, beta=1.0, mv=True)
        th_full = self.full_of(th)
        return (g_new, f_new, l_new, r_new, om_new, ns_new,
                Sharded(th_full.reshape(-1) if vec else th_full, True))

    def plain_richardson(self, theta: Sharded, p: Sharded, a: Sharded, b: Sharded) -> Sharded:
        """theta - P (A theta - b) with replicated theta/b; returns the
        gathered (replicated) new theta.  A vector theta/b (n,) is handled as n x 1."""
        vec = theta.t.ndim == 1
        if vec:
            theta = Sharded(theta.t.reshape(-1, 1), theta.full)
            b = Sharded(b.t.reshape(-1, 1), b.full)
        resid = self.mm(a, theta, c=b, beta=-1.0, mv=True)
        new = self.mm(p, resid, alpha=-1.0, c=theta, beta=1.0, mv=True)
        out = self.full_of(new)
        return Sharded(out.reshape(-1) if vec else out, True)


def _reads(ins, reg: str) -> bool:
    if isinstance(ins, Mul):
        return reg in (ins.lhs, ins.rhs)
    if isinstance(ins, Residual):
        return ins.src == reg
    return any(r == reg for _, r in ins.terms)
