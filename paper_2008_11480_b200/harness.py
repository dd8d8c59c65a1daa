"""Comparison runs over the device path: the caller side of the hot path
(per-step error norms, predicted bounds and CSV emission).

Mirrors the reference's ``run_comparison`` / ``RunRecord`` / CSV layer
(harness.py:163-404): every method is stepped through the B200 steps, the
per-step error norms are device reductions (``si_fro_norm``), the predicted
bound is rho^(e_k - e_0) err_0 with rho from the device power iteration, and
the CSV (17 significant digits) parses back to the same records.  The
injectable ``timer`` is called exactly as the reference calls it (once per
method, then once per record), so a deterministic timer gives byte-identical
``wall_ns`` columns.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from . import _lib
from .matrix_core import (SpectralRadiusError, fro_norm, mat_vec, spectral_radius, square_matrix,
                          vector)
from .newton_schulz import (CompositeSpec, additive_correction_step, additive_exponents,
                            classical_exponent, composite_exponent, composite_step,
                            double_exponent, double_ns_step, initial_double, initial_series,
                            ns_step)
from .richardson import (cumulative_exponent, initial_richardson, richardson_recursive_step,
                         richardson_step)
from .series_toolkit import factored_mmm, split_candidates
from .splitting import split_scalar

__all__ = ["CSV_HEADER", "DIVERGENCE_FACTOR", "INVERSION_KINDS", "MethodSpec", "RunRecord",
           "parse_run_records", "records_to_csv", "run_comparison", "series_params"]

INVERSION_KINDS = ("ns", "double", "composite", "sri")          # hx:76
ESTIMATOR_KINDS = ("ns-estimator", "richardson", "richardson-recursive")
DIVERGENCE_FACTOR = 1e3                                          # hx:78
CSV_HEADER = "method,k,error_norm,predicted_bound,exponent,mmm_cum,wall_ns"  # hx:393


@dataclass(frozen=True)
class MethodSpec:
    """One method of a comparison run (hx:163-192): ``kind`` in INVERSION_KINDS
    (the inversion residual ||I - G A||_F is tracked) or ESTIMATOR_KINDS (the
    parameter mismatch ||theta - theta*|| is tracked)."""

    kind: str
    order: int = 2
    h: int = 1
    q: int | None = None
    rates: tuple[int, ...] = ()
    label: str | None = None

    def name(self) -> str:
        if self.label:
            return self.label
        if self.kind == "composite":
            return f"composite:n{self.order}:h{self.h}:r{'-'.join(map(str, self.rates))}"
        if self.kind == "sri":
            return f"sri:p{self.order}:h{self.h}"
        if self.kind in ("richardson", "richardson-recursive"):
            return f"{self.kind}:n{self.order}:q{self.order if self.q is None else self.q}:h{self.h}"
        return f"{self.kind}:n{self.order}:h{self.h}"


@dataclass
class RunRecord:
    """One (method, step) measurement (hx:195-210); ``diverged`` is not a CSV
    column."""

    method: str
    k: int
    error_norm: float
    predicted_bound: float
    exponent: int
    mmm_cum: int
    wall_ns: int
    diverged: bool = field(default=False, compare=False)


def series_params(h: int) -> tuple[int, int]:
    """Cheapest (p, w) with w (p + 1) = h for the initial series (hx:213-224)."""
    if h < 1:
        raise ValueError("h must be >= 1")
    if h == 1:
        return 0, 1
    best = (h - 1, 1)
    for cand in split_candidates(h):
        if factored_mmm(*cand) < factored_mmm(*best):
            best = cand
    return best


def _rho(split) -> float:
    try:
        return spectral_radius(split.residual, tol=1e-10, max_iter=20000)
    except SpectralRadiusError as exc:
        return exc.best_estimate


def _residual_norm(g, a) -> float:
    """||I - G A||_F for measurement only (no MulCounter tick), on the device."""
    out = torch.empty_like(g)
    _lib.call("si_gemm", _lib.handle(g.device.index), g.shape[0], a.shape[1], g.shape[1], -1.0,
              g.data_ptr(), g.shape[1], a.data_ptr(), a.shape[1], 0.0, None, a.shape[1], 1.0,
              out.data_ptr(), a.shape[1], 0, None, _lib.stream_ptr(g.device))
    return fro_norm(out)


def _mismatch(theta, theta_star) -> float:
    return fro_norm(theta.reshape(-1) - theta_star.reshape(-1))


def _inversion_states(m: MethodSpec, split, a, steps):
    p, w = series_params(m.h)
    n = m.order
    if m.kind in ("ns", "composite"):
        if m.kind == "composite" and not m.rates:
            raise ValueError("composite method needs rates")
        spec = CompositeSpec(rates=m.rates) if m.kind == "composite" else None
        st = initial_series(split, p, w, order=n)
        yield 0, fro_norm(st.residual), st.ctr.mmm
        for _ in range(steps):
            st = ns_step(st, a) if spec is None else composite_step(st, a, split, spec, order_n=n)
            yield st.step, fro_norm(st.residual), st.ctr.mmm
    elif m.kind == "double":
        st = initial_double(split, p, w, order=n)
        yield 0, fro_norm(st.residual), st.ctr.mmm
        for _ in range(steps):
            st = double_ns_step(st, a)
            yield st.step, fro_norm(st.residual), st.ctr.mmm
    elif m.kind == "sri":
        st = initial_series(split, p, w, order=n)
        z = g = st.estimate
        ctr = st.ctr
        yield 0, fro_norm(st.residual), ctr.mmm
        for k in range(1, steps + 1):
            z, g = additive_correction_step(z, g, a, n, ctr)
            yield k, _residual_norm(g, a), ctr.mmm   # measured off the counter
    else:
        raise ValueError(f"unknown inversion kind {m.kind!r}")


def _estimator_states(m: MethodSpec, split, a, b, theta_star, steps):
    p, w = series_params(m.h)
    n = m.order
    if m.kind == "ns-estimator":
        st = initial_series(split, p, w, order=n)
        theta = mat_vec(st.estimate, b, st.ctr)
        yield 0, _mismatch(theta, theta_star), st.ctr.mmm
        for _ in range(steps):
            st = ns_step(st, a)
            theta = mat_vec(st.estimate, b, st.ctr)
            yield st.step, _mismatch(theta, theta_star), st.ctr.mmm
    elif m.kind in ("richardson", "richardson-recursive"):
        st = initial_richardson(split, b, p, w, order=n, q=m.q)
        yield 0, _mismatch(st.theta, theta_star), st.ctr.mmm
        step = richardson_step if m.kind == "richardson" else richardson_recursive_step
        for _ in range(steps):
            st = step(st, a, b)
            yield st.step, _mismatch(st.theta, theta_star), st.ctr.mmm
    else:
        raise ValueError(f"unknown estimator kind {m.kind!r}")


def _exponent(m: MethodSpec, k: int) -> int:
    n, h = m.order, m.h
    if m.kind in ("ns", "ns-estimator"):
        return classical_exponent(k, n, h)
    if m.kind == "double":
        return double_exponent(k, n, h)
    if m.kind == "composite":
        return composite_exponent(k, n, h, m.rates)
    if m.kind == "sri":
        return additive_exponents(k, n, h)[1]
    if m.kind in ("richardson", "richardson-recursive"):
        return cumulative_exponent(k, n, h, n if m.q is None else m.q)
    raise ValueError(f"unknown kind {m.kind!r}")


def _run_method(m: MethodSpec, split, a, b, theta_star, steps, rho, timer) -> list[RunRecord]:
    started = timer()
    states = (_inversion_states(m, split, a, steps) if m.kind in INVERSION_KINDS
              else _estimator_states(m, split, a, b, theta_star, steps))
    out: list[RunRecord] = []
    err0 = None
    e0 = _exponent(m, 0)
    for k, err, mmm in states:
        if err0 is None:
            err0 = err
        e = _exponent(m, k)
        out.append(RunRecord(method=m.name(), k=k, error_norm=err,
                             predicted_bound=rho ** (e - e0) * err0, exponent=e, mmm_cum=mmm,
                             wall_ns=int(timer() - started),
                             diverged=bool(err > DIVERGENCE_FACTOR * max(err0, 1e-300))))
    return out


def run_comparison(a, b, theta_star, methods: list[MethodSpec], steps: int, *,
                   eps: float | None = None, timer=None, executor=None) -> list[RunRecord]:
    """Every method for ``steps`` steps on one scalar splitting (hx:343-387);
    records sorted by (method, k).  With ``executor`` the methods run
    concurrently (the library handle is shared and thread-safe) and the merged
    records equal the serial run's."""
    a = square_matrix(a)
    b = vector(b)
    theta_star = vector(theta_star)
    if steps < 0:
        raise ValueError("steps must be >= 0")
    if timer is None:
        timer = time.perf_counter_ns
    split = split_scalar(a, eps)
    rho = _rho(split)
    if executor is None:
        chunks = [_run_method(m, split, a, b, theta_star, steps, rho, timer) for m in methods]
    else:
        futs = [executor.submit(_run_method, m, split, a, b, theta_star, steps, rho, timer)
                for m in methods]
        chunks = [f.result() for f in futs]
    merged = [r for c in chunks for r in c]
    merged.sort(key=lambda r: (r.method, r.k))
    return merged


def records_to_csv(records: list[RunRecord]) -> str:
    """CSV with 17 significant digits so parsing round-trips (hx:395-404)."""
    rows = [CSV_HEADER]
    rows += [f"{r.method},{r.k},{r.error_norm:.16e},{r.predicted_bound:.16e},{r.exponent},"
             f"{r.mmm_cum},{r.wall_ns}" for r in records]
    return "\n".join(rows) + "\n"


def parse_run_records(text: str) -> list[RunRecord]:
    """Inverse of :func:`records_to_csv` (hx:407-423)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != CSV_HEADER:
        raise ValueError("missing or unexpected CSV header")
    out = []
    for ln in lines[1:]:
        f = ln.split(",")
        if len(f) != 7:
            raise ValueError(f"bad record line: {ln!r}")
        out.append(RunRecord(method=f[0], k=int(f[1]), error_norm=float(f[2]),
                             predicted_bound=float(f[3]), exponent=int(f[4]), mmm_cum=int(f[5]),
                             wall_ns=int(f[6])))
    return out

