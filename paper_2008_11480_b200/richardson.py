"""Parameter estimation A theta = b with the inversion accelerator (richardson.py).

Device-resident counterpart of ``seriesinv.richardson``: ``theta`` may be a
vector (n,) or a block of right-hand sides (n, r); the step bodies are single
C-ABI calls.  ``plain_richardson`` is the north_star's update
theta + P (b - A theta) with products ordered as richardson.py:88-89.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .matrix_core import MulCounter, as_device
from .newton_schulz import DoubleNsState, initial_double
from .series_toolkit import FactorPlan, encode_plan
from .splitting import Splitting

__all__ = [
    "RichardsonState",
    "TransientModel",
    "cumulative_exponent",
    "cumulative_exponent_closed",
    "initial_richardson",
    "plain_richardson",
    "richardson_recursive_step",
    "richardson_step",
    "step_exponent_general",
    "step_exponent_qn",
    "transient_model",
]


@dataclass
class RichardsonState:
    """theta_k plus the two-loop inversion state (richardson.py:42-58)."""

    theta: torch.Tensor
    inner: DoubleNsState
    q: int
    omega: torch.Tensor | None
    ns_part: torch.Tensor | None
    step: int
    ctr: MulCounter


def _rhs(t: torch.Tensor) -> tuple[torch.Tensor, int]:
    t2 = t.reshape(t.shape[0], -1).contiguous()
    return t2, t2.shape[1]


def initial_richardson(split: Splitting, b, p: int = 0, w: int = 1, order: int = 2,
                       q: int | None = None) -> RichardsonState:
    """theta_0 = L_0 b (richardson.py:61-78)."""
    inner = initial_double(split, p, w, order)
    if q is None:
        q = order
    if q < 1:
        raise ValueError("q must be >= 1")
    b = as_device(b)
    b2, r = _rhs(b)
    theta = torch.empty_like(b2)
    n = b2.shape[0]
    buf = _lib.counter_buf()
    _lib.call("si_gemm", _lib.handle(b.device.index), n, r, n, 1.0, inner.accel_estimate.data_ptr(),
              n, b2.data_ptr(), r, 0.0, None, r, 0.0, theta.data_ptr(), r, 1, buf,
              _lib.stream_ptr(b.device))
    inner.ctr.absorb(buf)
    return RichardsonState(theta=theta.reshape(b.shape), inner=inner, q=q, omega=None, ns_part=None,
                           step=0, ctr=inner.ctr)


def _check(st: RichardsonState, a: torch.Tensor, b: torch.Tensor):
    if a.shape[0] != st.theta.shape[0] or tuple(b.shape) != tuple(st.theta.shape):
        raise ValueError("dimension mismatch")


def richardson_step(st: RichardsonState, a, b) -> RichardsonState:
    """Direct form (richardson.py:81-98)."""
    a, b = as_device(a), as_device(b)
    _check(st, a, b)
    inner = st.inner
    b2, r = _rhs(b)
    th2, _ = _rhs(st.theta)
    g, f, l, rr = (torch.empty_like(inner.estimate) for _ in range(4))
    theta = torch.empty_like(th2)
    buf = _lib.counter_buf()
    _lib.call("si_richardson_step", _lib.handle(a.device.index), a.shape[0], r, a.data_ptr(),
              b2.data_ptr(), th2.data_ptr(), inner.estimate.data_ptr(), inner.residual.data_ptr(),
              inner.accel_estimate.data_ptr(), inner.accel_residual.data_ptr(), inner.order, st.q,
              g.data_ptr(), f.data_ptr(), l.data_ptr(), rr.data_ptr(), theta.data_ptr(), buf,
              _lib.stream_ptr(a.device))
    st.ctr.absorb(buf)
    new_inner = DoubleNsState(estimate=g, residual=f, accel_estimate=l, accel_residual=rr,
                              step=inner.step + 1, order=inner.order,
                              series_order=inner.series_order, ctr=st.ctr)
    return RichardsonState(theta=theta.reshape(st.theta.shape), inner=new_inner, q=st.q, omega=None,
                           ns_part=None, step=st.step + 1, ctr=st.ctr)


_RECURSIVE_INPUTS = ("a", "b", "theta", "estimate", "residual", "accel_estimate",
                     "accel_residual", "omega", "ns_part")
_RECURSIVE_OUTPUTS = ("accel_estimate", "accel_residual", "estimate", "residual", "ns_part",
                      "omega", "theta")


def _event_array(events: dict | None, names: tuple, what: str, recorded: bool):
    if not events:
        return None
    unknown = set(events) - set(names)
    if unknown:
        raise ValueError(f"unknown names in {what}: {sorted(unknown)}")
    return (ctypes.c_void_p * len(names))(
        *[_lib.event_ptr(events.get(k), recorded=recorded) for k in names])


def richardson_recursive_step(st: RichardsonState, a, b, executor=None, *,
                              factor_plan: FactorPlan | None = None,
                              doubling_sum: bool = False, inputs_ready: dict | None = None,
                              outputs_done: dict | None = None) -> RichardsonState:
    """Recursive form, q == n only (richardson.py:111-189).

    Opt-in (not in the reference; changes the GEMM count): ``factor_plan`` of
    order n evaluates N' through a factorised plan and ``doubling_sum``
    builds S = prod (I + Gamma^(2^j)) for power-of-two n.

    Host-copy overlap (``si_richardson_recursive_step_ex``): ``inputs_ready``
    maps input names (``a``, ``b``, ``theta`` and the state fields) to CUDA
    events recorded behind their host->device copies -- the step waits for an
    input right before its first use; ``outputs_done`` maps the new state's
    field names to events the step records once that field is final."""
    n = st.inner.order
    if st.q != n:
        raise ValueError("the recursive form requires q == n")
    a, b = as_device(a), as_device(b)
    _check(st, a, b)
    if factor_plan is not None and factor_plan.order_h != n:
        raise ValueError(f"plan order {factor_plan.order_h} != iteration order {n}")
    if doubling_sum and (n < 2 or n & (n - 1)):
        raise ValueError("doubling_sum requires a power-of-two order")
    code, consts = encode_plan(factor_plan) if factor_plan is not None else ([], [])
    prev = st.inner
    b2, r = _rhs(b)
    th2, _ = _rhs(st.theta)
    g, f, l, rr, om, nsp = (torch.empty_like(prev.estimate) for _ in range(6))
    theta = torch.empty_like(th2)
    buf = _lib.counter_buf()
    ready = _event_array(inputs_ready, _RECURSIVE_INPUTS, "inputs_ready", True)
    done = _event_array(outputs_done, _RECURSIVE_OUTPUTS, "outputs_done", False)
    _lib.call("si_richardson_recursive_step_ex", _lib.handle(a.device.index), a.shape[0], r,
              a.data_ptr(), b2.data_ptr(), th2.data_ptr(), prev.estimate.data_ptr(),
              prev.residual.data_ptr(), prev.accel_estimate.data_ptr(),
              prev.accel_residual.data_ptr(), _lib.ptr(st.omega), _lib.ptr(st.ns_part), n,
              _lib.i32_array(code) if code else None, len(code),
              _lib.f64_array(consts) if consts else None, len(consts), int(doubling_sum),
              int(executor is not None), ready, done, g.data_ptr(), f.data_ptr(), l.data_ptr(),
              rr.data_ptr(), om.data_ptr(), nsp.data_ptr(), theta.data_ptr(), buf,
              _lib.stream_ptr(a.device))
    st.ctr.absorb(buf)
    inner = DoubleNsState(estimate=g, residual=f, accel_estimate=l, accel_residual=rr,
                          step=prev.step + 1, order=n, series_order=prev.series_order, ctr=st.ctr)
    return RichardsonState(theta=theta.reshape(st.theta.shape), inner=inner, q=st.q, omega=om,
                           ns_part=nsp, step=st.step + 1, ctr=st.ctr)


def plain_richardson(theta, p, a, b, ctr: MulCounter) -> torch.Tensor:
    """theta + P (b - A theta), as theta - P (A theta - b) (richardson.py:88-89)."""
    theta, p, a, b = as_device(theta), as_device(p), as_device(a), as_device(b)
    if a.shape[0] != theta.shape[0] or tuple(b.shape) != tuple(theta.shape):
        raise ValueError("dimension mismatch")
    b2, r = _rhs(b)
    th2, _ = _rhs(theta)
    out = torch.empty_like(th2)
    buf = _lib.counter_buf()
    _lib.call("si_plain_richardson", _lib.handle(a.device.index), a.shape[0], r, a.data_ptr(),
              b2.data_ptr(), th2.data_ptr(), p.data_ptr(), out.data_ptr(), buf,
              _lib.stream_ptr(a.device))
    ctr.absorb(buf)
    return out.reshape(theta.shape)


# ---------------------------------------------------------------------------
# Transient models (richardson.py:197-266): integer host arithmetic
# ---------------------------------------------------------------------------


def step_exponent_general(k: int, n: int, h: int, q: int) -> int:
    return h * ((k * n ** (k + 1) + n**k) * q + n ** (k + 1))


def step_exponent_qn(k: int, n: int, h: int) -> int:
    return h * (k * n ** (k + 2) + 2 * n ** (k + 1))


def cumulative_exponent(k: int, n: int, h: int, q: int | None = None) -> int:
    if q is None or q == n:
        return sum(step_exponent_qn(j, n, h) for j in range(1, k + 1))
    return sum(step_exponent_general(j, n, h, q) for j in range(1, k + 1))


def cumulative_exponent_closed(k: int, n: int, h: int) -> int:
    if n < 2:
        raise ValueError("closed form requires n >= 2")
    if k < 1 or h < 1:
        raise ValueError("requires k >= 1 and h >= 1")
    num = h * n * n * (k * n ** (k + 2) - (k - 1) * n ** (k + 1) - 2 * n**k - n + 2)
    quo, rem = divmod(num, (n - 1) ** 2)
    if rem:
        raise ArithmeticError(f"closed form not divisible: {num} / {(n - 1) ** 2}")
    return quo


@dataclass(frozen=True)
class TransientModel:
    total_exponent: int
    step_exponent: int
    rho: float
    bound: float


def transient_model(k: int, n: int, h: int, rho: float, q: int | None = None,
                    theta0_norm: float = 1.0) -> TransientModel:
    if k < 1:
        raise ValueError("transient model starts at step 1")
    step = step_exponent_qn(k, n, h) if (q is None or q == n) else step_exponent_general(k, n, h, q)
    total = cumulative_exponent(k, n, h, q)
    return TransientModel(total, step, rho, float(rho) ** total * theta0_norm)
