"""High-order Newton-Schulz family on the device (newton_schulz.py).

Same signatures, state fields and errors as ``seriesinv.newton_schulz``; the
states hold device tensors and every step body is one C-ABI call that runs the
reference's GEMM DAG on the DMMA kernels.  ``executor`` arguments map to
concurrent CUDA streams (bitwise identical to the serial path).  The integer
exponent laws (newton_schulz.py:343-400) are host arithmetic and are restated
here unchanged in meaning.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from math import sqrt

import torch

from . import _lib
from .matrix_core import MulCounter, as_device, fro_norm
from .series_toolkit import FactorPlan, encode_many, encode_plan, geometric_base_plan
from .splitting import Splitting

__all__ = [
    "CompositeParts",
    "CompositeSpec",
    "composite_parts",
    "DoubleNsState",
    "NsState",
    "additive_correction_step",
    "additive_exponents",
    "classical_exponent",
    "composite_exponent",
    "composite_step",
    "constant_rates",
    "converged",
    "double_exponent",
    "double_ns_step",
    "initial_double",
    "initial_series",
    "ns_step",
    "power_rates",
    "residual_exponent",
    "run_until_converged",
]

DEFAULT_MAX_STEPS = 30


def _step_call(name: str, h, like: torch.Tensor, *args) -> torch.Tensor:
    """One step call with its residual's ||F'||_F^2 fused into the products
    that write F' (si_set_step_norm, a one-shot target); returns that device
    double."""
    fro2 = torch.empty(1, dtype=torch.float64, device=like.device)
    _lib.call("si_set_step_norm", h, fro2.data_ptr())
    try:
        _lib.call(name, h, *args)
    except BaseException:
        _lib.call("si_set_step_norm", h, None)
        raise
    return fro2


@dataclass
class NsState:
    """G_k (estimate), F_k = I - G_k A (residual) (newton_schulz.py:58-72)."""

    estimate: torch.Tensor
    residual: torch.Tensor
    step: int
    order: int
    series_order: int
    ctr: MulCounter
    # ||F_k||_F^2 as a device double, fused into the epilogues of the products
    # that wrote F_k (si_set_step_norm); read by converged()
    residual_fro2: torch.Tensor | None = field(default=None, compare=False, repr=False)


@dataclass
class DoubleNsState:
    """Two-loop state with accelerator L_k and its residual (newton_schulz.py:75-91)."""

    estimate: torch.Tensor
    residual: torch.Tensor
    accel_estimate: torch.Tensor
    accel_residual: torch.Tensor
    step: int
    order: int
    series_order: int
    ctr: MulCounter
    residual_fro2: torch.Tensor | None = field(default=None, compare=False, repr=False)


@dataclass(frozen=True)
class CompositeSpec:
    """Expansion rates x_i, one per parallel unit (newton_schulz.py:94-108)."""

    rates: tuple[int, ...]

    def __post_init__(self):
        if not self.rates:
            raise ValueError("composite spec needs at least one rate")
        if any(x < 1 for x in self.rates):
            raise ValueError("rates must be positive integers")

    @property
    def width(self) -> int:
        return len(self.rates)


def constant_rates(rate: int, width: int) -> CompositeSpec:
    return CompositeSpec(rates=(rate,) * width)


def power_rates(base: int, width: int):
    """At step k every unit expands at rate base**k (newton_schulz.py:116-124)."""
    if base < 2:
        raise ValueError("base must be >= 2")

    def spec_for_step(k: int) -> CompositeSpec:
        return CompositeSpec(rates=(base**k,) * width)

    return spec_for_step


def _ctx(t: torch.Tensor):
    return _lib.handle(t.device.index), _lib.stream_ptr(t.device)


def initial_series(split: Splitting, p: int, w: int, order: int = 2) -> NsState:
    """G_0 = S_h(B) S^-1 with h = w(p+1) (newton_schulz.py:127-147)."""
    if order < 1:
        raise ValueError("order must be >= 1")
    if p < 0 or w < 1:
        raise ValueError("requires p >= 0 and w >= 1")
    ctr = MulCounter()
    n = split.matrix.shape[0]
    g = torch.empty_like(split.matrix)
    f = torch.empty_like(split.matrix)
    h, s = _ctx(g)
    buf = _lib.counter_buf()
    nrm = _step_call("si_initial_series", h, g, n, split.precond.data_ptr(),
                     split.residual.data_ptr(), split.matrix.data_ptr(), p, w, g.data_ptr(),
                     f.data_ptr(), buf, s)
    ctr.absorb(buf)
    return NsState(estimate=g, residual=f, step=0, order=order, series_order=w * (p + 1), ctr=ctr,
                   residual_fro2=nrm)


def ns_step(st: NsState, a, plan: FactorPlan | None = None, *, inputs_ready: dict | None = None,
            estimate_done=None, input_panels: tuple | None = None,
            residual_chunks: list | None = None) -> NsState:
    """G_k = S_n(F) G (Horner or ``plan``), F_k = I - G_k A (newton_schulz.py:150-174).

    ``inputs_ready`` (keys ``a``, ``estimate``, ``residual``), ``estimate_done``,
    ``input_panels`` (flags 3 x 16 for a, estimate, residual) and
    ``residual_chunks`` as in :func:`composite_step`."""
    n = st.order
    a = as_device(a)
    if a.shape != st.estimate.shape:
        raise ValueError("dimension mismatch between state and matrix")
    code: list[int] = []
    consts: list[float] = []
    if plan is not None:
        if plan.order_h != n:
            raise ValueError(f"plan order {plan.order_h} != iteration order {n}")
        code, consts = encode_plan(plan)
    g = torch.empty_like(st.estimate)
    f = torch.empty_like(st.estimate)
    h, s = _ctx(g)
    buf = _lib.counter_buf()
    if input_panels is not None or residual_chunks:
        if inputs_ready:
            raise ValueError("inputs_ready and input_panels are exclusive")
        flags_ptr, epoch, npanels = _panel_args(input_panels, 48)
        chunks = list(residual_chunks or [])
        evs = (ctypes.c_void_p * max(len(chunks), 1))(*[_lib.event_ptr(e) for e in chunks])
        nrm = _step_call("si_ns_step_gated", h, g, a.shape[0], a.data_ptr(), st.estimate.data_ptr(),
                         st.residual.data_ptr(), n, _lib.i32_array(code) if code else None,
                         len(code), _lib.f64_array(consts) if consts else None, len(consts),
                         flags_ptr, epoch, npanels,
                         _lib.event_ptr(estimate_done),
                         evs if chunks else None, len(chunks), g.data_ptr(), f.data_ptr(), buf, s)
        st.ctr.absorb(buf)
        return NsState(estimate=g, residual=f, step=st.step + 1, order=n,
                       series_order=st.series_order, ctr=st.ctr, residual_fro2=nrm)
    ready = None
    if inputs_ready:
        order3 = ("a", "estimate", "residual")
        unknown = set(inputs_ready) - set(order3)
        if unknown:
            raise ValueError(f"unknown inputs in inputs_ready: {sorted(unknown)}")
        ready = (ctypes.c_void_p * 3)(
            *[_lib.event_ptr(inputs_ready.get(k), recorded=True) for k in order3])
    nrm = _step_call("si_ns_step_ex", h, g, a.shape[0], a.data_ptr(), st.estimate.data_ptr(),
                     st.residual.data_ptr(), n, _lib.i32_array(code) if code else None, len(code),
                     _lib.f64_array(consts) if consts else None, len(consts), ready,
                     _lib.event_ptr(estimate_done), g.data_ptr(),
                     f.data_ptr(), buf, s)
    st.ctr.absorb(buf)
    return NsState(estimate=g, residual=f, step=st.step + 1, order=n,
                   series_order=st.series_order, ctr=st.ctr, residual_fro2=nrm)


def _panel_args(input_panels, words: int):
    """(flags pointer, epoch, npanels) of an ``input_panels`` tuple (or Nones)."""
    if input_panels is None:
        return None, 0, 0
    flags, epoch, npanels = input_panels
    if flags.dtype != torch.int32 or flags.numel() < words or not flags.is_cuda:
        raise ValueError(f"input_panels flags must be a CUDA int32 tensor of {words} flags")
    if not 1 <= npanels <= 16:
        raise ValueError("npanels must be in 1..16")
    return flags.data_ptr(), epoch, npanels


@dataclass
class CompositeParts:
    """Hoisted state-independent half of the composite step (opt-in; the
    reference recomputes it every step): T_comp and R_comp (newton_schulz.py:204-216)."""

    t_comp: torch.Tensor
    r_comp: torch.Tensor
    rates: tuple[int, ...]


def composite_parts(a, split: Splitting, spec: CompositeSpec, ctr: MulCounter) -> CompositeParts:
    """Evaluate the parts T_i, Gamma_i and their left fold once (opt-in hoisting)."""
    a = as_device(a)
    plans = [geometric_base_plan(x) if x > 1 else None for x in spec.rates]
    code, offsets, consts = encode_many(plans)
    t = torch.empty_like(a)
    r = torch.empty_like(a)
    h, s = _ctx(a)
    buf = _lib.counter_buf()
    _lib.call("si_composite_parts", h, a.shape[0], a.data_ptr(), split.precond.data_ptr(),
              split.residual.data_ptr(), split.matrix.data_ptr(), len(spec.rates),
              _lib.i32_array(list(spec.rates)), _lib.i32_array(code), _lib.i64_array(offsets),
              _lib.f64_array(consts), len(consts), t.data_ptr(), r.data_ptr(), buf, s)
    ctr.absorb(buf)
    return CompositeParts(t_comp=t, r_comp=r, rates=tuple(spec.rates))


_READY_ORDER = ("a", "estimate", "residual", "precond", "split_residual", "matrix")


def composite_step(st: NsState, a, split: Splitting, spec: CompositeSpec, order_n: int,
                   executor=None, parts: CompositeParts | None = None, *,
                   inputs_ready: dict | None = None, estimate_done=None,
                   input_panels: tuple | None = None,
                   residual_chunks: list | None = None) -> NsState:
    """G_k = T_comp + R_comp S_n(F) G, F_k = I - G_k A (newton_schulz.py:177-228).

    ``executor`` (not in the reference signature, whose parts run serially)
    evaluates the independent parts on concurrent streams.  ``parts`` (opt-in,
    changes the GEMM count) reuses hoisted T_comp / R_comp from
    :func:`composite_parts` instead of recomputing them.

    ``inputs_ready`` maps input names (``a``, ``estimate``, ``residual``,
    ``precond``, ``split_residual``, ``matrix``) to recorded ``torch.cuda.Event``s
    (e.g. host->device copies on another stream); the step waits on each right
    before that input's first use.  ``estimate_done`` is recorded when the new
    estimate is final, before the last product.

    ``input_panels = (flags, epoch, npanels)`` instead: the inputs arrive in row
    panels; ``flags`` is a CUDA int32 tensor of 6 x 16 flags (inputs a,
    estimate, residual, precond, split_residual, matrix; panel p of n rows is
    rows [n p / npanels, n (p+1) / npanels)), raised (>= epoch) behind each
    panel's copy -- the products gate their loads per panel.  The flags must be
    raised by work that needs no SM (copy-engine copies, stream memory
    operations): the gated products may hold every SM while they wait.
    ``residual_chunks`` (list of ``torch.cuda.Event``): G' and F' are produced
    in that many row blocks, interleaved (G' block k, then F' block k), each
    event recorded once both blocks are final -- both may go device->host
    while the next blocks are computed; ``estimate_done`` then fires when the
    last G' block is final."""
    if order_n < 1:
        raise ValueError("order_n must be >= 1")
    a = as_device(a)
    if a.shape != st.estimate.shape:
        raise ValueError("dimension mismatch between state and matrix")
    if parts is not None:
        if tuple(parts.rates) != tuple(spec.rates):
            raise ValueError("hoisted parts were built for different rates")
        g = torch.empty_like(st.estimate)
        f = torch.empty_like(st.estimate)
        h, s = _ctx(g)
        buf = _lib.counter_buf()
        nrm = _step_call("si_composite_apply", h, g, a.shape[0], a.data_ptr(),
                         st.estimate.data_ptr(), st.residual.data_ptr(), parts.t_comp.data_ptr(),
                         parts.r_comp.data_ptr(), order_n, g.data_ptr(), f.data_ptr(), buf, s)
        st.ctr.absorb(buf)
        return NsState(estimate=g, residual=f, step=st.step + 1, order=order_n,
                       series_order=st.series_order, ctr=st.ctr, residual_fro2=nrm)
    plans = [geometric_base_plan(x) if x > 1 else None for x in spec.rates]
    code, offsets, consts = encode_many(plans)
    g = torch.empty_like(st.estimate)
    f = torch.empty_like(st.estimate)
    h, s = _ctx(g)
    buf = _lib.counter_buf()
    if input_panels is not None or residual_chunks:
        if inputs_ready:
            raise ValueError("inputs_ready and input_panels are exclusive")
        flags_ptr, epoch, npanels = _panel_args(input_panels, 96)
        chunks = list(residual_chunks or [])
        evs = (ctypes.c_void_p * max(len(chunks), 1))(*[_lib.event_ptr(e) for e in chunks])
        nrm = _step_call("si_composite_step_gated", h, g, a.shape[0], a.data_ptr(),
                         st.estimate.data_ptr(), st.residual.data_ptr(), split.precond.data_ptr(),
                         split.residual.data_ptr(), split.matrix.data_ptr(), len(spec.rates),
                         _lib.i32_array(list(spec.rates)), _lib.i32_array(code),
                         _lib.i64_array(offsets), _lib.f64_array(consts), len(consts), order_n,
                         int(executor is not None), flags_ptr, epoch, npanels,
                         _lib.event_ptr(estimate_done),
                         evs if chunks else None, len(chunks), g.data_ptr(), f.data_ptr(), buf, s)
        st.ctr.absorb(buf)
        return NsState(estimate=g, residual=f, step=st.step + 1, order=order_n,
                       series_order=st.series_order, ctr=st.ctr, residual_fro2=nrm)
    ready = None
    if inputs_ready:
        unknown = set(inputs_ready) - set(_READY_ORDER)
        if unknown:
            raise ValueError(f"unknown inputs in inputs_ready: {sorted(unknown)}")
        ready = (ctypes.c_void_p * len(_READY_ORDER))(
            *[_lib.event_ptr(inputs_ready.get(k), recorded=True) for k in _READY_ORDER])
    nrm = _step_call("si_composite_step_ex", h, g, a.shape[0], a.data_ptr(), st.estimate.data_ptr(),
                     st.residual.data_ptr(), split.precond.data_ptr(), split.residual.data_ptr(),
                     split.matrix.data_ptr(), len(spec.rates), _lib.i32_array(list(spec.rates)),
                     _lib.i32_array(code), _lib.i64_array(offsets), _lib.f64_array(consts),
                     len(consts), order_n, int(executor is not None), ready,
                     _lib.event_ptr(estimate_done), g.data_ptr(),
                     f.data_ptr(), buf, s)
    st.ctr.absorb(buf)
    return NsState(estimate=g, residual=f, step=st.step + 1, order=order_n,
                   series_order=st.series_order, ctr=st.ctr, residual_fro2=nrm)


def initial_double(split: Splitting, p: int, w: int, order: int = 2) -> DoubleNsState:
    """Two-loop init: L_0 = S_n(F_0) G_0 (newton_schulz.py:231-251)."""
    if order < 1:
        raise ValueError("order must be >= 1")
    if p < 0 or w < 1:
        raise ValueError("requires p >= 0 and w >= 1")
    ctr = MulCounter()
    m = split.matrix
    g, f, l, r = (torch.empty_like(m) for _ in range(4))
    h, s = _ctx(m)
    buf = _lib.counter_buf()
    nrm = _step_call("si_initial_double", h, m, m.shape[0], split.precond.data_ptr(),
                     split.residual.data_ptr(), m.data_ptr(), p, w, order, g.data_ptr(),
                     f.data_ptr(), l.data_ptr(), r.data_ptr(), buf, s)
    ctr.absorb(buf)
    return DoubleNsState(estimate=g, residual=f, accel_estimate=l, accel_residual=r, step=0,
                         order=order, series_order=w * (p + 1), ctr=ctr, residual_fro2=nrm)


def double_ns_step(st: DoubleNsState, a, executor=None) -> DoubleNsState:
    """F_k = (I - L_k A) F_(k-1)^n (newton_schulz.py:254-298); ``executor`` -> two streams."""
    a = as_device(a)
    if a.shape != st.estimate.shape:
        raise ValueError("dimension mismatch between state and matrix")
    g, f, l, r = (torch.empty_like(st.estimate) for _ in range(4))
    h, s = _ctx(g)
    buf = _lib.counter_buf()
    nrm = _step_call("si_double_ns_step", h, g, a.shape[0], a.data_ptr(), st.estimate.data_ptr(),
                     st.residual.data_ptr(), st.accel_estimate.data_ptr(),
                     st.accel_residual.data_ptr(), st.order, int(executor is not None),
                     g.data_ptr(), f.data_ptr(), l.data_ptr(), r.data_ptr(), buf, s)
    st.ctr.absorb(buf)
    return DoubleNsState(estimate=g, residual=f, accel_estimate=l, accel_residual=r,
                         step=st.step + 1, order=st.order, series_order=st.series_order,
                         ctr=st.ctr, residual_fro2=nrm)


def additive_correction_step(z, g, a, p: int, ctr: MulCounter):
    """Two-estimate additive scheme (newton_schulz.py:301-325)."""
    if p < 2:
        raise ValueError("order p must be >= 2")
    z, g, a = as_device(z), as_device(g), as_device(a)
    zn = torch.empty_like(z)
    gn = torch.empty_like(g)
    h, s = _ctx(z)
    buf = _lib.counter_buf()
    _lib.call("si_additive_correction_step", h, a.shape[0], a.data_ptr(), z.data_ptr(),
              g.data_ptr(), p, zn.data_ptr(), gn.data_ptr(), buf, s)
    ctr.absorb(buf)
    return zn, gn


def converged(st) -> bool:
    """||F_k||_F <= 1e-13 sqrt(n) (newton_schulz.py:328-331)."""
    dim = st.residual.shape[0]
    fro2 = getattr(st, "residual_fro2", None)
    norm = sqrt(float(fro2.item())) if fro2 is not None else fro_norm(st.residual)
    return norm <= 1e-13 * sqrt(dim)


def run_until_converged(st: NsState, a, max_steps: int = DEFAULT_MAX_STEPS) -> NsState:
    """Classical steps until converged or the cap (newton_schulz.py:334-340)."""
    while st.step < max_steps and not converged(st):
        st = ns_step(st, a)
    return st


# ---------------------------------------------------------------------------
# Integer exponent laws: F_k = B**e (newton_schulz.py:343-400)
# ---------------------------------------------------------------------------


def classical_exponent(k: int, n: int, h: int) -> int:
    return h * n**k


def double_exponent(k: int, n: int, h: int) -> int:
    return h * (k * n ** (k + 1) + n**k)


def composite_exponent(k: int, n: int, h: int, rates: tuple[int, ...]) -> int:
    e, total = h, sum(rates)
    for _ in range(k):
        e = total + n * e
    return e


def additive_exponents(k: int, p: int, h: int) -> tuple[int, int]:
    e_l = e_f = h
    for _ in range(k):
        e_f += p * e_l
        e_l *= p
    return e_l, e_f


def residual_exponent(kind: str, k: int, n: int, h: int, rates=None) -> int:
    if k < 0:
        raise ValueError("step index must be >= 0")
    if kind == "classical":
        return classical_exponent(k, n, h)
    if kind == "double":
        return double_exponent(k, n, h)
    if kind == "composite":
        if not rates:
            raise ValueError("composite kind needs rates")
        return composite_exponent(k, n, h, tuple(rates))
    if kind == "additive":
        return additive_exponents(k, n, h)[1]
    raise ValueError(f"unknown iteration kind: {kind!r}")
