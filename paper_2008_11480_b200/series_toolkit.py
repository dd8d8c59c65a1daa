"""Plans and evaluators for ``S_h(Y) X = (I + Y + ... + Y^(h-1)) X``.

Host side: the plan vocabulary of ``seriesinv.series_toolkit`` (series_toolkit.py:
71-157, FactorPlan/make_plan/plan_str :160-255, the catalogue :465-664, the
search :682-747) -- small integer trees, chosen once per run and lowered to an
int32 preorder code (``encode_plan``) that the native engine executes.

Device side: ``horner_eval`` / ``factored_eval`` / ``nested_eval`` /
``geometric_apply`` call the C ABI; every product runs on the DMMA GEMM with
its element-wise follow-up fused in the epilogue.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache
from typing import Union

import torch

from . import _lib
from .matrix_core import MulCounter, as_device

__all__ = [
    "FactorPlan",
    "Horner",
    "Lin",
    "Mul",
    "PrimeWrap",
    "Residual",
    "Split",
    "TABLE_LABELS",
    "TableForm",
    "efficiency_index",
    "encode_plan",
    "factored_eval",
    "factored_mmm",
    "geometric_apply",
    "geometric_base_order",
    "horner_eval",
    "make_plan",
    "nested_eval",
    "order45_plan",
    "plan_order",
    "plan_str",
    "split_candidates",
    "table_plans",
]

MAX_PLAN_ORDER = 64
_MAX_NESTING = 3

# ---------------------------------------------------------------------------
# Node vocabulary (series_toolkit.py:71-157)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Horner:
    order: int


@dataclass(frozen=True)
class Split:
    p: int
    w: int
    inner: "PlanNode"
    outer: "PlanNode | None" = None


@dataclass(frozen=True)
class PrimeWrap:
    inner: "PlanNode"


@dataclass(frozen=True)
class Mul:
    dst: str
    lhs: str
    rhs: str


@dataclass(frozen=True)
class Residual:
    dst: str
    src: str


@dataclass(frozen=True)
class Lin:
    dst: str
    const: float
    terms: tuple[tuple[float, str], ...]


Instr = Union[Mul, Residual, Lin]


@dataclass(frozen=True)
class TableForm:
    label: str
    order: int
    program: tuple[Instr, ...]


PlanNode = Union[Horner, Split, PrimeWrap, TableForm]


@dataclass(frozen=True)
class FactorPlan:
    order_h: int
    root: PlanNode
    mmm_cost: int
    mmm_poly: int
    efficiency_index: float


def _order(node) -> int:
    """Order of a node, validating the tree (series_toolkit.py:165-192)."""
    if isinstance(node, Horner):
        if node.order < 1:
            raise ValueError("Horner order must be >= 1")
        return node.order
    if isinstance(node, Split):
        if node.p < 0 or node.w < 1:
            raise ValueError("Split requires p >= 0 and w >= 1")
        if node.p >= 1 and _order(node.inner) != node.p + 1:
            raise ValueError(f"Split inner order {_order(node.inner)} != p + 1 = {node.p + 1}")
        if node.w >= 2:
            if node.outer is None:
                raise ValueError("Split with w >= 2 needs an outer node")
            if _order(node.outer) != node.w:
                raise ValueError(f"Split outer order {_order(node.outer)} != w = {node.w}")
        return node.w * (node.p + 1)
    if isinstance(node, PrimeWrap):
        return _order(node.inner) + 1
    if isinstance(node, TableForm):
        return node.order
    raise TypeError(f"not a plan node: {node!r}")


def _poly(node) -> int:
    """Products with Y supplied (series_toolkit.py:195-207)."""
    if isinstance(node, Horner):
        return node.order - 1
    if isinstance(node, Split):
        c = 0 if node.p == 0 else _poly(node.inner)
        if node.w >= 2:
            c += (0 if node.p == 0 else 1) + _poly(node.outer)
        return c
    if isinstance(node, PrimeWrap):
        return _poly(node.inner) + 1
    if isinstance(node, TableForm):
        return sum(isinstance(i, (Mul, Residual)) for i in node.program)
    raise TypeError(f"not a plan node: {node!r}")


def _depth(node) -> int:
    if isinstance(node, Horner):
        return 0
    if isinstance(node, Split):
        return 1 + max(_depth(node.inner), _depth(node.outer) if node.outer is not None else 0)
    if isinstance(node, PrimeWrap):
        return _depth(node.inner)
    if isinstance(node, TableForm):
        return 1
    raise TypeError(f"not a plan node: {node!r}")


def make_plan(root: PlanNode) -> FactorPlan:
    """Validate and attach counts (series_toolkit.py:224-237)."""
    order = _order(root)
    poly = _poly(root)
    return FactorPlan(order, root, poly + 1, poly, float(order) ** (1.0 / (poly + 1)))


def plan_str(plan) -> str:
    """Canonical one-line form (series_toolkit.py:240-255)."""
    node = plan.root if isinstance(plan, FactorPlan) else plan
    if isinstance(node, Horner):
        return f"horner(h={node.order})"
    if isinstance(node, Split):
        bits = [f"p={node.p},w={node.w}"]
        if node.p >= 1 and not isinstance(node.inner, Horner):
            bits.append(f"inner={plan_str(node.inner)}")
        if node.w >= 2 and node.outer is not None and not isinstance(node.outer, Horner):
            bits.append(f"outer={plan_str(node.outer)}")
        return "split(" + ", ".join(bits) + ")"
    if isinstance(node, PrimeWrap):
        return f"wrap({plan_str(node.inner)})"
    if isinstance(node, TableForm):
        return f"table({node.label})"
    raise TypeError(f"not a plan node: {node!r}")


def factored_mmm(p: int, w: int) -> int:
    """Full-step count of the two-level split (series_toolkit.py:305-317)."""
    if p < 0 or w < 1:
        raise ValueError("requires p >= 0 and w >= 1")
    if w == 1:
        return p + 1
    if p == 0:
        return w
    return p + w + 1


def efficiency_index(p: int, w: int) -> float:
    """Order per product ``(w(p+1))**(1/count)`` (series_toolkit.py:320-323)."""
    return float(w * (p + 1)) ** (1.0 / factored_mmm(p, w))


# ---------------------------------------------------------------------------
# Catalogue (series_toolkit.py:465-664).  The folded forms are written in a
# compact text DSL:  "d=a*b" product, "d=r(s)" residual I - s A,
# "d=c+x+y" sum with constant c times I.
# ---------------------------------------------------------------------------

_FORM_SOURCE = {
    "h5b": (5, "y2=Y*Y s=0+Y+y2 t=y2*s m=1+Y+y2+t z=m*X"),
    "h7": (7, "y2=Y*Y y4=y2*y2 f1=0+Y+y4 f2=1+Y+y2 w=f1*f2 t=w*X z=0+X+t"),
    "h8": (8, "c0=Y*X c1=0+X+c0 q2=r(c1) c2=q2*c1 c3=0+c1+c2 q4=r(c3) c4=q4*c3 z=0+c3+c4"),
    "h9b": (9, "y2=Y*Y y4=y2*y2 f1=0+Y+y2 f2=1+y2 w1=f2*f1 f3=1+y4 w2=f3*w1 t=w2*X z=0+X+t"),
    "h10b": (10, "y2=Y*Y f1=0+Y+y2 f2=1+y2 w=f1*f2 t0=w*X u=0+X+t0 q5=r(u) t1=q5*u z=0+u+t1"),
    "h11b": (11, "t0=Y*X t1=0+X+t0 y2=r(t1) y4=y2*y2 f1=0+y2+y4 f2=1+y4 w=f1*f2 t2=w*t1 "
                 "t3=0+t1+t2 t4=Y*t3 z=0+X+t4"),
    "h15b": (15, "c0=Y*X c1=0+X+c0 c2=Y*c1 u=0+X+c2 q3=r(u) q6=q3*q3 f1=1+q6 f2=0+q3+q6 "
                 "w=f1*f2 t=w*u z=0+u+t"),
    "h17": (17, "y2=Y*Y f1=0+Y+y2 f2=1+y2 g=f1*f2 y4=y2*y2 y8=y4*y4 y12=y8*y4 "
                "f3=1+y4+y8+y12 w=g*f3 t=w*X z=0+X+t"),
    "h19": (19, "y2=Y*Y y4=y2*y2 f1=0+Y+y2 f2=1+y2+y4 w1=f1*f2 y6=y2*y4 y12=y6*y6 "
                "f3=1+y6+y12 w2=w1*f3 t=w2*X z=0+X+t"),
}


def _parse_form(label: str) -> TableForm:
    order, src = _FORM_SOURCE[label]
    prog: list[Instr] = []
    for stmt in src.split():
        dst, rhs = stmt.split("=")
        if rhs.startswith("r(") and rhs.endswith(")"):
            prog.append(Residual(dst, rhs[2:-1]))
        elif "*" in rhs:
            lhs, r = rhs.split("*")
            prog.append(Mul(dst, lhs, r))
        else:
            const, *regs = rhs.split("+")
            prog.append(Lin(dst, float(const), tuple((1.0, r) for r in regs)))
    return TableForm(label=label, order=order, program=tuple(prog))


_FORMS = {label: _parse_form(label) for label in _FORM_SOURCE}


def _unit_split(p: int, w: int) -> Split:
    return Split(p, w, Horner(p + 1), Horner(w) if w >= 2 else None)


_CATALOGUE: dict[int, tuple[tuple[str, PlanNode], ...]] = {
    2: (("h2", _unit_split(1, 1)),),
    3: (("h3", PrimeWrap(_unit_split(1, 1))),),
    4: (("h4", _unit_split(1, 2)),),
    5: (("h5a", PrimeWrap(_unit_split(1, 2))), ("h5b", _FORMS["h5b"])),
    6: (("h6", _unit_split(2, 2)),),
    7: (("h7", _FORMS["h7"]),),
    8: (("h8", _FORMS["h8"]),),
    9: (("h9a", _unit_split(2, 3)), ("h9b", _FORMS["h9b"])),
    10: (("h10a", PrimeWrap(_unit_split(2, 3))), ("h10b", _FORMS["h10b"])),
    11: (("h11a", PrimeWrap(_FORMS["h10b"])), ("h11b", _FORMS["h11b"])),
    12: (("h12", _unit_split(3, 3)),),
    13: (("h13", PrimeWrap(_unit_split(3, 3))),),
    14: (("h14", _unit_split(6, 2)),),
    15: (("h15a", _unit_split(2, 5)), ("h15b", _FORMS["h15b"])),
    16: (("h16", _unit_split(3, 4)),),
    17: (("h17", _FORMS["h17"]),),
    18: (("h18", _unit_split(5, 3)),),
    19: (("h19", _FORMS["h19"]),),
}

TABLE_LABELS: dict[int, tuple[str, ...]] = {
    order: tuple(label for label, _ in rows) for order, rows in _CATALOGUE.items()
}


@lru_cache(maxsize=1)
def table_plans() -> dict[int, list[FactorPlan]]:
    """Catalogued plans for orders 2..19 (series_toolkit.py:658-664)."""
    return {order: [make_plan(node) for _, node in rows] for order, rows in _CATALOGUE.items()}


def order45_plan() -> FactorPlan:
    """Order 45 in ten products (series_toolkit.py:667-676)."""
    return make_plan(Split(8, 5, Split(2, 3, Horner(3), Horner(3)), _FORMS["h5b"]))


def split_candidates(h: int) -> list[tuple[int, int]]:
    """(p, w) with w (p+1) == h, p >= 1, w >= 2 (series_toolkit.py:684-686)."""
    return [(d - 1, h // d) for d in range(2, h // 2 + 1) if h % d == 0]


def _prime(n: int) -> bool:
    return n >= 2 and all(n % d for d in range(2, int(n**0.5) + 1))


@lru_cache(maxsize=None)
def _search(h: int, budget: int):
    """Minimal (cost, rank, p, depth) node; ranks split < wrap < table < horner
    (series_toolkit.py:697-735)."""
    best = (h - 1, 3, 1 << 30, 0, Horner(h))
    options = [best]
    if budget >= 1:
        options += [(_poly(n), 2, 1 << 30, _depth(n), n) for _, n in _CATALOGUE.get(h, ())]
        if h == 2:
            options.append((1, 0, 1, 1, Split(1, 1, Horner(2))))
        for p, w in split_candidates(h):
            ic, _, _, idp, inner = _search(p + 1, budget - 1)
            oc, _, _, odp, outer = _search(w, budget - 1)
            options.append((ic + 1 + oc, 0, p, 1 + max(idp, odp), Split(p, w, inner, outer)))
        if h >= 3 and _prime(h):
            ic, _, _, idp, inner = _search(h - 1, budget)
            options.append((ic + 1, 1, 1 << 30, idp, PrimeWrap(inner)))
    return min(options, key=lambda o: o[:4])


def plan_order(h: int) -> FactorPlan:
    """Minimal-count plan for 2 <= h <= 64 (series_toolkit.py:738-747)."""
    if h < 2:
        raise ValueError("plan_order requires h >= 2")
    if h > MAX_PLAN_ORDER:
        raise ValueError(f"plan_order supports h <= {MAX_PLAN_ORDER}")
    return make_plan(_search(h, _MAX_NESTING)[4])


# ---------------------------------------------------------------------------
# Lowering to the native int32 preorder code
# ---------------------------------------------------------------------------


class _Encoder:
    def __init__(self):
        self.code: list[int] = []
        self.consts: list[float] = []

    def const(self, v: float) -> int:
        v = float(v)
        for i, c in enumerate(self.consts):
            if c == v:
                return i
        self.consts.append(v)
        return len(self.consts) - 1

    def node(self, n) -> None:
        if isinstance(n, Horner):
            self.code += [0, n.order]
        elif isinstance(n, Split):
            self.code += [1, n.p, n.w]
            for child in (n.inner, n.outer):
                if child is None:
                    self.code.append(0)
                else:
                    self.code.append(1)
                    self.node(child)
        elif isinstance(n, PrimeWrap):
            self.code.append(2)
            self.node(n.inner)
        elif isinstance(n, TableForm):
            regs = {"Y": 0, "X": 1}

            def reg(name: str) -> int:
                if name not in regs:
                    regs[name] = len(regs)
                return regs[name]

            body: list[int] = []
            for ins in n.program:
                if isinstance(ins, Mul):
                    body += [0, reg(ins.dst), reg(ins.lhs), reg(ins.rhs)]
                elif isinstance(ins, Residual):
                    body += [1, reg(ins.dst), reg(ins.src)]
                elif isinstance(ins, Lin):
                    body += [2, reg(ins.dst), self.const(ins.const), len(ins.terms)]
                    for coef, r in ins.terms:
                        body += [self.const(coef), reg(r)]
                else:
                    raise TypeError(f"bad instruction {ins!r}")
            self.code += [3, n.order, len(regs), len(n.program)] + body
        else:
            raise TypeError(f"not a plan node: {n!r}")


def encode_plan(plan) -> tuple[list[int], list[float]]:
    """FactorPlan / node -> (int32 preorder code, constant pool)."""
    node = plan.root if isinstance(plan, FactorPlan) else plan
    enc = _Encoder()
    enc.node(node)
    return enc.code, enc.consts


def encode_many(nodes) -> tuple[list[int], list[int], list[float]]:
    """Concatenate several plans (None -> empty) with a shared constant pool."""
    enc = _Encoder()
    offsets = [0]
    for n in nodes:
        if n is not None:
            enc.node(n.root if isinstance(n, FactorPlan) else n)
        offsets.append(len(enc.code))
    return enc.code, offsets, enc.consts


def geometric_base_order(order: int) -> int:
    """The order <= 64 geometric_apply bottoms out at (series_toolkit.py:449-457)."""
    while order > MAX_PLAN_ORDER:
        order //= 2
    return order


def geometric_base_plan(order: int) -> FactorPlan | None:
    b = geometric_base_order(order)
    return plan_order(b) if b >= 2 else None


# ---------------------------------------------------------------------------
# Device evaluators (series_toolkit.py:279-457)
# ---------------------------------------------------------------------------


def _dev_args(x, a=None, y=None):
    x = as_device(x)
    a = as_device(a) if a is not None else None
    y = as_device(y) if y is not None else None
    return x, a, y


def horner_eval(y, x, h: int, ctr: MulCounter, *, a=None, form_y: bool = False) -> torch.Tensor:
    """``S_h(Y) X`` by Horner; h-1 products, h with form_y (series_toolkit.py:279-302)."""
    if h < 1:
        raise ValueError("order h must be >= 1")
    if form_y and a is None:
        raise ValueError("form_y=True requires the matrix a")
    if not form_y and y is None:
        raise ValueError("y is required unless form_y=True")
    x, a, y = _dev_args(x, a, y)
    out = torch.empty_like(x)
    buf = _lib.counter_buf()
    _lib.call("si_horner_eval", _lib.handle(x.device.index), x.shape[0], _lib.ptr(y), x.data_ptr(),
              h, _lib.ptr(a), int(form_y), out.data_ptr(), buf, _lib.stream_ptr(x.device))
    ctr.absorb(buf)
    return out


def factored_eval(y, x, a, p: int, w: int, ctr: MulCounter, *, form_y: bool = True) -> torch.Tensor:
    """Two-level factored evaluation of order w(p+1) (series_toolkit.py:326-356)."""
    if p < 0 or w < 1:
        raise ValueError("requires p >= 0 and w >= 1")
    x, a, y = _dev_args(x, a, y)
    if x.shape != a.shape:
        raise ValueError(f"dimension mismatch: x {tuple(x.shape)} vs a {tuple(a.shape)}")
    if not form_y and y is None:
        raise ValueError("y is required unless form_y=True")
    out = torch.empty_like(x)
    buf = _lib.counter_buf()
    _lib.call("si_factored_eval", _lib.handle(x.device.index), x.shape[0], _lib.ptr(y),
              x.data_ptr(), a.data_ptr(), p, w, int(form_y), out.data_ptr(), buf,
              _lib.stream_ptr(x.device))
    ctr.absorb(buf)
    return out


def nested_eval(y, x, a, plan: FactorPlan, ctr: MulCounter, *, form_y: bool = True) -> torch.Tensor:
    """Execute a plan; counter moves by mmm_cost (mmm_poly with form_y=False)
    (series_toolkit.py:408-429)."""
    if _order(plan.root) != plan.order_h:
        raise ValueError("malformed plan: order does not match its tree")
    x, a, y = _dev_args(x, a, y)
    if x.shape != a.shape:
        raise ValueError(f"dimension mismatch: x {tuple(x.shape)} vs a {tuple(a.shape)}")
    if not form_y and y is None:
        raise ValueError("y is required unless form_y=True")
    code, consts = encode_plan(plan)
    out = torch.empty_like(x)
    buf = _lib.counter_buf()
    _lib.call("si_nested_eval", _lib.handle(x.device.index), x.shape[0], _lib.ptr(y), x.data_ptr(),
              a.data_ptr(), _lib.i32_array(code), len(code), _lib.f64_array(consts), len(consts),
              int(form_y), out.data_ptr(), buf, _lib.stream_ptr(x.device))
    ctr.absorb(buf)
    return out


def geometric_apply(y, x, order: int, a, ctr: MulCounter) -> torch.Tensor:
    """``S_order(Y) X`` for any order, Y supplied (series_toolkit.py:432-457)."""
    if order < 1:
        raise ValueError("order must be >= 1")
    x, a, y = _dev_args(x, a, y)
    base = geometric_base_plan(order)
    code, consts = encode_plan(base) if base is not None else ([], [])
    out = torch.empty_like(x)
    buf = _lib.counter_buf()
    _lib.call("si_geometric_apply", _lib.handle(x.device.index), x.shape[0], y.data_ptr(),
              x.data_ptr(), order, a.data_ptr(), _lib.i32_array(code) if code else None, len(code),
              _lib.f64_array(consts) if consts else None, len(consts), out.data_ptr(), buf,
              _lib.stream_ptr(x.device))
    ctr.absorb(buf)
    return out
