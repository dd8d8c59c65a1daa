"""The CUDA library as a ``cases`` backend (device tensors in, numpy out)."""

from __future__ import annotations

import numpy as np
import torch

import paper_2008_11480_b200 as P


class GpuBackend:
    name = "gpu"

    def __init__(self, concurrent: bool = False):
        self.concurrent = concurrent
        self.executor = object() if concurrent else None

    def counter(self):
        return P.MulCounter()

    def np(self, x):
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy()
        return np.asarray(x)

    def dev(self, x):
        return P.as_device(x)

    def plan_order(self, h):
        return P.plan_order(h)

    def table_plan(self, order, idx):
        return P.table_plans()[order][idx]

    def table_items(self):
        for order, plans in P.table_plans().items():
            for label, plan in zip(P.TABLE_LABELS[order], plans):
                yield order, label, plan

    def order45(self):
        return P.order45_plan()

    def mat_mul(self, a, b, c):
        return P.mat_mul(a, b, c)

    def mat_pow_counted(self, y, e, c):
        return P.mat_pow_counted(y, e, c)

    def horner_eval(self, y, x, h, c, a=None, form_y=False):
        return P.horner_eval(y, x, h, c, a=a, form_y=form_y)

    def factored_eval(self, y, x, a, p, w, c, form_y):
        return P.factored_eval(y, x, a, p, w, c, form_y=form_y)

    def nested_eval(self, y, x, a, plan, c, form_y=True):
        return P.nested_eval(y, x, a, plan, c, form_y=form_y)

    def geometric_apply(self, y, x, order, a, c):
        return P.geometric_apply(y, x, order, a, c)

    def split_scalar(self, a, eps):
        return P.split_scalar(a, eps)

    def split_diagonal(self, a):
        return P.split_diagonal(a)

    def initial_series(self, sp, p, w, order):
        return P.initial_series(sp, p, w, order=order)

    def ns_step(self, st, a, plan=None):
        return P.ns_step(st, a, plan=plan)

    def composite_step(self, st, a, sp, rates, n):
        return P.composite_step(st, a, sp, P.CompositeSpec(tuple(rates)), n, executor=self.executor)

    def initial_double(self, sp, p, w, order):
        return P.initial_double(sp, p, w, order=order)

    def double_ns_step(self, st, a):
        return P.double_ns_step(st, a, executor=self.executor)

    def additive(self, z, g, a, p, c):
        return P.additive_correction_step(z, g, a, p, c)

    def initial_richardson(self, sp, b, p, w, order, q):
        return P.initial_richardson(sp, b, p, w, order=order, q=q)

    def richardson_step(self, st, a, b):
        return P.richardson_step(st, a, b)

    def richardson_recursive_step(self, st, a, b):
        return P.richardson_recursive_step(st, a, b, executor=self.executor)

    def plain(self, theta, p, a, b, c):
        return P.plain_richardson(theta, p, a, b, c)

    def inf_norm(self, a):
        return P.inf_norm(a)

