"""BASELINE configs 2 and 3 at full size against the live oracle, and the step
entry points' concurrency / inputs-in-flight variants.  (The full-length
config-4 / config-5 runs against the oracle are at n=4096 and config 4 at its
full size in test_gpu_fullsize.py.)"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _kappa_tol(a, tol=1e-10):
    ev = np.linalg.eigvalsh(a)
    return tol * max(1.0, float(ev.max() / ev.min()) / 1e4)


def test_c3_full_size_25_iterations_vs_oracle():
    """BASELINE config 3 exactly (n=4096, Gram 8192x4096, h8 plan + plain Richardson,
    25 iterations): P_k and theta_k against the live oracle at every iteration."""
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    a, b = configs.c3_gram(n=4096)
    tol = _kappa_tol(a)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    st = P.initial_series(sp, 0, 1, order=8)
    bd = P.as_device(b)
    theta = torch.zeros_like(bd)
    osp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    ost = O.initial_series(osp, 0, 1, 8)
    oth = np.zeros_like(b)
    plan, oplan = P.table_plans()[8][0], O.TABLE_ROOTS[8][0][1]
    worst = 0.0
    for k in range(25):
        theta = P.plain_richardson(theta, st.estimate, sp.matrix, bd, st.ctr)
        st = P.ns_step(st, sp.matrix, plan=plan)
        oth = O.plain_richardson(oth, ost.estimate, osp.matrix, b, ost.ctr)
        ost = O.ns_step(ost, osp.matrix, oplan)
        ep = np.linalg.norm(st.estimate.cpu().numpy() - ost.estimate) / np.linalg.norm(ost.estimate)
        et = np.linalg.norm(theta.cpu().numpy() - oth) / np.linalg.norm(oth)
        worst = max(worst, ep, et)
        assert ep <= tol and et <= tol, (k, ep, et)
    assert (st.ctr.mmm, st.ctr.mvm) == (ost.ctr.mmm, ost.ctr.mvm) == (150, 50)
    print(f"c3 full size: worst rel err {worst:.3e}")


def test_c2_full_batch_sampled_vs_oracle():
    """BASELINE config 2 exactly (16384 systems, 50 iterations, one launch); 48 sampled
    systems against the oracle."""
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    a_np, b_np = configs.c2_batched(batch=16384)
    a, b = P.as_device(a_np), P.as_device(b_np)
    pre, res = P.batched_scalar_split(a)
    ctr = P.MulCounter()
    p, f, th = P.batched_composite_richardson(a, b, pre, res, pre, res, torch.zeros_like(b),
                                              (2, 3), 2, 50, ctr)
    assert (ctr.mmm, ctr.mvm) == (500, 100)  # per system: 10 + 2 per iteration
    for i in np.random.default_rng(7).choice(16384, 48, replace=False):
        sp = O.split_scalar(a_np[i], O.inf_norm(a_np[i]) / 2.0)
        st = O.initial_series(sp, 0, 1, 2)
        theta = np.zeros(32)
        for _ in range(50):
            theta = O.plain_richardson(theta, st.estimate, sp.matrix, b_np[i], st.ctr)
            st = O.composite_step(st, sp.matrix, sp, (2, 3), 2)
        assert np.linalg.norm(p[i].cpu().numpy() - st.estimate) <= 1e-10 * np.linalg.norm(st.estimate)
        assert np.linalg.norm(th[i].cpu().numpy() - theta) <= 1e-10 * np.linalg.norm(theta)


def test_host_threads_share_the_handle():
    """The reference runs methods from executor threads (harness.py:371-380): steps
    issued concurrently from several host threads give bitwise the serial results."""
    from concurrent.futures import ThreadPoolExecutor

    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a, b = configs.c4_householder(n=384, rhs=4)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    bd = P.as_device(b)

    def run(kind):
        torch.cuda.set_device(0)
        if kind == "composite":
            st = P.initial_series(sp, 0, 1, order=2)
            for _ in range(3):
                st = P.composite_step(st, sp.matrix, sp, P.CompositeSpec((2, 3, 4, 5)), 2)
            out = st.estimate
        elif kind == "double":
            st = P.initial_double(sp, 1, 2, order=3)
            for _ in range(3):
                st = P.double_ns_step(st, sp.matrix, executor=True)
            out = st.estimate
        else:
            st = P.initial_richardson(sp, bd, 0, 1, order=4, q=4)
            for _ in range(3):
                st = P.richardson_recursive_step(st, sp.matrix, bd, executor=True)
            out = st.theta
        torch.cuda.current_stream().synchronize()
        return out.clone()

    kinds = ["composite", "double", "recursive"] * 2
    serial = [run(k) for k in kinds]
    with ThreadPoolExecutor(max_workers=3) as pool:
        threaded = list(pool.map(run, kinds))
    for s, t in zip(serial, threaded):
        assert torch.equal(s, t)


def test_composite_step_with_inputs_in_flight():
    """Inputs copied host->device on another stream, the step waiting on per-input
    events: bitwise the same result as with resident inputs."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a, _ = configs.c4_householder(n=768, rhs=1)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    spec = P.CompositeSpec((2, 3, 4, 5))
    st = P.initial_series(sp, 0, 1, order=2)
    ref = P.composite_step(st, sp.matrix, sp, spec, 2)
    host = {k: v.cpu().pin_memory() for k, v in (("a", sp.matrix), ("p", sp.precond),
                                                   ("b", sp.residual), ("g", st.estimate),
                                                   ("f", st.residual))}
    up = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    up.wait_stream(main)
    d, ev = {}, {}
    with torch.cuda.stream(up):
        for k in ("p", "b", "a", "g", "f"):
            d[k] = host[k].to("cuda", non_blocking=True)
            d[k].record_stream(main)
            ev[k] = torch.cuda.Event()
            ev[k].record(up)
    sp2 = P.Splitting(precond=d["p"], residual=d["b"], matrix=d["a"], kind="scalar", verify=False)
    st2 = P.NsState(estimate=d["g"], residual=d["f"], step=0, order=2, series_order=1,
                    ctr=P.MulCounter())
    done = torch.cuda.Event()
    out = P.composite_step(st2, sp2.matrix, sp2, spec, 2, inputs_ready={
        "precond": ev["p"], "split_residual": ev["b"], "matrix": ev["a"], "a": ev["a"],
        "estimate": ev["g"], "residual": ev["f"]}, estimate_done=done)
    done.synchronize()
    assert torch.equal(out.estimate, ref.estimate)
    torch.cuda.synchronize()
    assert torch.equal(out.residual, ref.residual)
    with pytest.raises(ValueError):
        P.composite_step(st, sp.matrix, sp, spec, 2, inputs_ready={"bogus": done})


@pytest.mark.parametrize("backend,concurrent,n,npanels", [
    ("dmma", False, 768, 6), ("dmma", True, 768, 6), ("ozaki", False, 768, 6),
    ("ozaki", True, 768, 6), ("ozaki", False, 4096, 2)])
def test_composite_step_with_inputs_in_row_panels(backend, concurrent, n, npanels):
    """Inputs copied host->device panel by panel (out of order, a delaying copy
    first) with flags; the DMMA products gate their loads per panel (the
    emulated products wait per row chunk of A and for whole B / C operands) and
    F' comes out in row blocks: bitwise the resident-input result, same product
    count.  n=4096 with 2048-row panels: the emulated first product runs in row
    chunks behind the copy of its left operand."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib, configs

    if backend == "ozaki":
        # every product emulated, the F' row blocks (192 rows) included
        P.set_gemm_backend("ozaki", 16, 128)
    try:
        _inputs_in_row_panels(P, _lib, configs, concurrent, n, npanels)
    finally:
        P.set_gemm_backend("dmma", 16, 1024)


def _inputs_in_row_panels(P, _lib, configs, concurrent, n, npanels):
    a, _ = configs.c4_householder(n=n, rhs=1)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    spec = P.CompositeSpec((2, 3, 4, 5))
    st = P.initial_series(sp, 0, 1, order=2)
    c0 = st.ctr.mmm
    ref = P.composite_step(st, sp.matrix, sp, spec, 2)
    n_ref = ref.ctr.mmm - c0
    host = {k: v.cpu().pin_memory() for k, v in (("a", sp.matrix), ("p", sp.precond),
                                                   ("b", sp.residual), ("g", st.estimate),
                                                   ("f", st.residual))}
    flags = torch.zeros(96, dtype=torch.int32, device="cuda")
    slot = {"a": (0, 5), "g": (1,), "f": (2,), "p": (3,), "b": (4,)}
    d = {k: torch.empty_like(v, device="cuda") for k, v in host.items()}
    # the delay on the copy stream must not need SMs (the gated products may hold
    # them all while they wait): a host->device copy runs on a copy engine
    big = torch.empty(16 << 20, dtype=torch.float64).pin_memory()
    big2 = torch.empty(big.shape, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    up = torch.cuda.Stream()
    h = _lib.handle(0)
    bounds = [n * p // npanels for p in range(npanels + 1)]
    st2 = P.NsState(estimate=d["g"], residual=d["f"], step=0, order=2, series_order=1,
                    ctr=P.MulCounter())
    sp2 = P.Splitting(precond=d["p"], residual=d["b"], matrix=d["a"], kind="scalar", verify=False)
    chunks = [torch.cuda.Event() for _ in range(4)]
    done = torch.cuda.Event()
    # G' / F' read back row block by row block behind the events the step
    # records (the host buffers exist before the call: pinned allocation
    # synchronises the device and would hide an ungated read-back)
    back_g = torch.zeros(n, n, dtype=torch.float64).pin_memory()
    back_f = torch.zeros(n, n, dtype=torch.float64).pin_memory()
    down = torch.cuda.Stream()
    out = P.composite_step(st2, sp2.matrix, sp2, spec, 2, object() if concurrent else None,
                           input_panels=(flags, 3, npanels), residual_chunks=chunks,
                           estimate_done=done)
    assert all(e.cuda_event for e in chunks) and done.cuda_event  # created, not lazy nulls
    cb = [n * k // len(chunks) for k in range(len(chunks) + 1)]
    for k, e in enumerate(chunks):
        down.wait_event(e)
        with torch.cuda.stream(down):
            back_g[cb[k]:cb[k + 1]].copy_(out.estimate[cb[k]:cb[k + 1]], non_blocking=True)
            back_f[cb[k]:cb[k + 1]].copy_(out.residual[cb[k]:cb[k + 1]], non_blocking=True)
    with torch.cuda.stream(up):
        big2.copy_(big, non_blocking=True)  # the step is already waiting on the flags
        for k in ("b", "p", "a", "g", "f"):
            for p in reversed(range(npanels)):
                r0, r1 = bounds[p], bounds[p + 1]
                d[k][r0:r1].copy_(host[k][r0:r1], non_blocking=True)
                for i in slot[k]:
                    _lib.call("si_stream_write_u32", h, flags.data_ptr() + 4 * (16 * i + p), 3,
                              up.cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(out.estimate, ref.estimate)
    assert torch.equal(out.residual, ref.residual)
    assert out.ctr.mmm == n_ref
    assert all(e.query() for e in chunks)
    assert torch.equal(back_g, ref.estimate.cpu()) and torch.equal(back_f, ref.residual.cpu())


def test_ns_step_with_inputs_in_flight():
    """ns_step (h8 plan and Horner) with A, G, F still being copied on another
    stream: waits on each input right before its first reader; bitwise equal."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a, _ = configs.c3_gram(n=640)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    plan8 = P.table_plans()[8][0]
    for order, plan in ((8, plan8), (3, None)):
        st = P.initial_series(sp, 0, 1, order=order)
        ref = P.ns_step(st, sp.matrix, plan=plan)
        host = {k: v.cpu().pin_memory() for k, v in (("a", sp.matrix), ("g", st.estimate),
                                                       ("f", st.residual))}
        up = torch.cuda.Stream()
        main = torch.cuda.current_stream()
        up.wait_stream(main)
        d, ev = {}, {}
        with torch.cuda.stream(up):
            for k in ("f", "g", "a"):
                d[k] = host[k].to("cuda", non_blocking=True)
                d[k].record_stream(main)
                ev[k] = torch.cuda.Event()
                ev[k].record(up)
        st2 = P.NsState(estimate=d["g"], residual=d["f"], step=0, order=order, series_order=1,
                        ctr=P.MulCounter())
        done = torch.cuda.Event()
        out = P.ns_step(st2, d["a"], plan=plan, inputs_ready={
            "a": ev["a"], "estimate": ev["g"], "residual": ev["f"]}, estimate_done=done)
        done.synchronize()
        assert torch.equal(out.estimate, ref.estimate)
        torch.cuda.synchronize()
        assert torch.equal(out.residual, ref.residual)
    with pytest.raises(ValueError):
        P.ns_step(st, sp.matrix, inputs_ready={"bogus": done})


def test_ns_step_with_inputs_in_row_panels():
    """ns_step (h8 plan) with F, G, A arriving in row panels behind flags and F'
    in row blocks: bitwise equal to resident inputs, same product count."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib, configs

    n, npanels = 640, 5
    a, _ = configs.c3_gram(n=n)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    plan8 = P.table_plans()[8][0]
    st = P.initial_series(sp, 0, 1, order=8)
    c0 = st.ctr.mmm
    ref = P.ns_step(st, sp.matrix, plan=plan8)
    n_ref = ref.ctr.mmm - c0
    host = {k: v.cpu().pin_memory() for k, v in (("a", sp.matrix), ("g", st.estimate),
                                                   ("f", st.residual))}
    d = {k: torch.empty_like(v, device="cuda") for k, v in host.items()}
    flags = torch.zeros(48, dtype=torch.int32, device="cuda")
    slot = {"a": 0, "g": 1, "f": 2}
    big = torch.empty(16 << 20, dtype=torch.float64).pin_memory()
    big2 = torch.empty(big.shape, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    up = torch.cuda.Stream()
    h = _lib.handle(0)
    bounds = [n * p // npanels for p in range(npanels + 1)]
    st2 = P.NsState(estimate=d["g"], residual=d["f"], step=0, order=8, series_order=1,
                    ctr=P.MulCounter())
    chunks = [torch.cuda.Event() for _ in range(3)]
    out = P.ns_step(st2, d["a"], plan=plan8, input_panels=(flags, 9, npanels),
                    residual_chunks=chunks)
    with torch.cuda.stream(up):
        big2.copy_(big, non_blocking=True)  # copy engine: the step waits on flags meanwhile
        for k in ("g", "f", "a"):
            for p in range(npanels):
                r0, r1 = bounds[p], bounds[p + 1]
                d[k][r0:r1].copy_(host[k][r0:r1], non_blocking=True)
                _lib.call("si_stream_write_u32", h, flags.data_ptr() + 4 * (16 * slot[k] + p), 9,
                          up.cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(out.estimate, ref.estimate)
    assert torch.equal(out.residual, ref.residual)
    assert out.ctr.mmm == n_ref


def test_hoisted_composite_parts_bitwise():
    """Opt-in hoisting evaluates the same T_comp / R_comp DAG once: the steps are
    bitwise identical to the reference-faithful recompute, at 3 products per step
    (order_n = 2) instead of 22."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import configs

    a, _ = configs.c4_householder(n=640, rhs=1)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    spec = P.CompositeSpec((2, 3, 4, 5))
    s1 = P.initial_series(sp, 0, 1, order=2)
    s2 = P.initial_series(sp, 0, 1, order=2)
    parts = P.composite_parts(sp.matrix, sp, spec, s2.ctr)
    assert s2.ctr.mmm == 19
    for _ in range(3):
        s1 = P.composite_step(s1, sp.matrix, sp, spec, 2)
        c0 = s2.ctr.mmm
        s2 = P.composite_step(s2, sp.matrix, sp, spec, 2, parts=parts)
        assert s2.ctr.mmm - c0 == 3
        assert torch.equal(s1.estimate, s2.estimate) and torch.equal(s1.residual, s2.residual)
    with pytest.raises(ValueError):
        P.composite_step(s2, sp.matrix, sp, P.CompositeSpec((2, 3)), 2, parts=parts)


def test_batched_composite_with_inputs_by_chunks():
    """Config-2 launch fed by chunks of systems (flags behind each chunk's
    copy, raised late and out of order) and read back per chunk on the done
    counters: bitwise the resident-input result."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib, configs

    batch, chunk = 1500, 400
    a_np, b_np = configs.c2_batched(batch=batch)
    a, b = P.as_device(a_np), P.as_device(b_np)
    pre, res = P.batched_scalar_split(a)
    t0 = torch.zeros_like(b)
    ref = P.batched_composite_richardson(a, b, pre, res, pre, res, t0, (2, 3), 2, 5)
    host = {k: v.cpu().pin_memory() for k, v in
            (("a", a), ("b", b), ("pre", pre), ("res", res), ("t", t0))}
    d = {k: torch.empty_like(v, device="cuda") for k, v in host.items()}
    nch = (batch + chunk - 1) // chunk
    flags = torch.zeros(nch, dtype=torch.int32, device="cuda")
    done = torch.zeros(nch, dtype=torch.int32, device="cuda")
    big = torch.empty(16 << 20, dtype=torch.float64).pin_memory()
    big2 = torch.empty(big.shape, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    up = torch.cuda.Stream()
    h = _lib.handle(0)
    out = P.batched_composite_richardson(d["a"], d["b"], d["pre"], d["res"], d["pre"], d["res"],
                                         d["t"], (2, 3), 2, 5, input_chunks=(flags, 4, chunk),
                                         chunk_done=done)
    with torch.cuda.stream(up):
        big2.copy_(big, non_blocking=True)  # copy engine delay: the kernel waits meanwhile
        for c in reversed(range(nch)):
            lo, hi = c * chunk, min(batch, (c + 1) * chunk)
            for k in d:
                d[k][lo:hi].copy_(host[k][lo:hi], non_blocking=True)
            _lib.call("si_stream_write_u32", h, flags.data_ptr() + 4 * c, 4, up.cuda_stream)
    torch.cuda.synchronize()
    for x, y in zip(out, ref):
        assert torch.equal(x, y)
    assert done.tolist() == [min(batch, (c + 1) * chunk) - c * chunk for c in range(nch)]
