"""FP64 products emulated on the INT8 tensor cores (Ozaki scheme II, csrc/ozaki.cu).

* the tcgen05 kind::i8 kernel alone is exact (integer products mod m_l),
* an emulated product meets its a-priori bound entry by entry and is at least
  as accurate as the DMMA product against an extended-precision reference,
* the fused epilogue (alpha, beta C in place, diag I at an offset), non-finite
  rows / columns, zero and extreme-magnitude rows,
* results are independent of the row split (bitwise) and deterministic,
* the hot-path steps (configs 3, 4, 5 recipes) under the emulated backend meet
  the north_star tolerance against the oracle at every iteration.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _restore_backend():
    import paper_2008_11480_b200 as P

    yield
    P.set_gemm_backend("dmma", 16, 1024)


def _pa_pb(k, nmod):
    import paper_2008_11480_b200 as P

    m = math.prod(P.ozaki_moduli(nmod))
    t = m.bit_length() - 1 - 2 - max(0, (k - 1).bit_length())
    return min(56, (t + 1) // 2), min(56, t // 2)


def _ozaki(a, b, nmod=16):
    import paper_2008_11480_b200 as P

    with P.gemm_backend("ozaki", moduli=nmod, min_dim=128):
        return P.mat_mul(a, b, P.MulCounter())


def _dmma(a, b):
    import paper_2008_11480_b200 as P

    with P.gemm_backend("dmma"):
        return P.mat_mul(a, b, P.MulCounter())


@pytest.mark.parametrize("kernel", ["pair", "single", "multicast"])
@pytest.mark.parametrize("planes,m,n,kp", [(1, 128, 256, 128), (3, 300, 520, 256),
                                           (2, 1000, 777, 1024), (16, 513, 300, 2048),
                                           (5, 129, 1000, 4096), (2, 1, 1, 128),
                                           (3, 1200, 257, 384)])
def test_int8_kernel_exact(planes, m, n, kp, kernel):
    """Both INT8 kernels (CTA pairs / single CTAs) reproduce the exact integer
    products mod m_l, ragged tiles (rows / columns past the 256 x 256 pair tile
    or the 128 x 256 tile, one-row / one-column products) included."""
    import paper_2008_11480_b200 as P

    mods = P.ozaki_moduli(16)
    g = torch.Generator(device="cuda").manual_seed(planes * 1000 + m)
    a = torch.randint(-128, 128, (planes, m, kp), dtype=torch.int8, device="cuda", generator=g)
    bt = torch.randint(-128, 128, (planes, n, kp), dtype=torch.int8, device="cuda", generator=g)
    P.set_ozaki_kernel(kernel)
    try:
        r = P.i8_gemm_mod(a, bt)
    finally:
        P.set_ozaki_kernel("auto")
    for l in range(planes):
        # |sum| <= kp * 2^14 < 2^53: the FP64 product of these integers is exact
        ref = torch.remainder(a[l].double() @ bt[l].double().T, mods[l]).to(torch.uint8)
        assert torch.equal(ref, r[l]), (l, int((ref != r[l]).sum()))


@pytest.mark.parametrize("planes,m,n,kp", [(3, 300, 512, 4096), (2, 257, 777, 2048),
                                           (16, 128, 256, 1024)])
def test_int8_kernel_k_ranges(planes, m, n, kp):
    """A long K runs as several launches of the single-CTA kernel, each later one
    adding the residues already stored before its reduction (si_ozaki_tune_ksplit,
    a tuning hook that is off by default): the same integers mod m_l for any
    range length, ragged column counts (byte path) included."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib

    mods = P.ozaki_moduli(16)
    g = torch.Generator(device="cuda").manual_seed(planes * 77 + kp)
    a = torch.randint(-128, 128, (planes, m, kp), dtype=torch.int8, device="cuda", generator=g)
    bt = torch.randint(-128, 128, (planes, n, kp), dtype=torch.int8, device="cuda", generator=g)
    P.set_ozaki_kernel("single")
    outs = []
    try:
        for ks in (0, 128, 512, 1536, 16384):
            _lib.call("si_ozaki_tune_ksplit", ks)
            outs.append(P.i8_gemm_mod(a, bt).clone())
    finally:
        _lib.call("si_ozaki_tune_ksplit", 0)
        P.set_ozaki_kernel("auto")
    for l in range(planes):
        ref = torch.remainder(a[l].double() @ bt[l].double().T, mods[l]).to(torch.uint8)
        for r in outs:
            assert torch.equal(ref, r[l]), l
    # and through a whole emulated product (K = 2048 in ranges of 512)
    rng = np.random.default_rng(3)
    x, y = (torch.from_numpy(rng.standard_normal((600, 2048))).cuda(),
            torch.from_numpy(rng.standard_normal((2048, 520))).cuda())
    whole = _ozaki(x, y)
    try:
        _lib.call("si_ozaki_tune_ksplit", 512)
        assert torch.equal(_ozaki(x, y), whole)
    finally:
        _lib.call("si_ozaki_tune_ksplit", 0)


def test_int8_kernel_extreme_residues():
    """All-(-128) operands: the largest int32 sums the kernel's reduction sees."""
    import paper_2008_11480_b200 as P

    mods = P.ozaki_moduli(4)
    a = torch.full((4, 256, 8192), -128, dtype=torch.int8, device="cuda")
    bt = torch.full((4, 256, 8192), -128, dtype=torch.int8, device="cuda")
    bt[:, ::2] = 127
    for kernel in ("pair", "single", "multicast"):
        P.set_ozaki_kernel(kernel)
        try:
            r = P.i8_gemm_mod(a, bt)
        finally:
            P.set_ozaki_kernel("auto")
        for l in range(4):
            ref = torch.remainder(a[l].double() @ bt[l].double().T, mods[l]).to(torch.uint8)
            assert torch.equal(ref, r[l])


def test_kernels_bitwise_on_emulated_products():
    """The emulated FP64 product is the same bits with either INT8 kernel."""
    import paper_2008_11480_b200 as P

    rng = np.random.default_rng(31)
    a = torch.from_numpy(rng.standard_normal((1500, 1300))).cuda()
    b = torch.from_numpy(rng.standard_normal((1300, 1700))).cuda()
    outs = []
    for kernel in ("pair", "single", "multicast"):
        P.set_ozaki_kernel(kernel)
        try:
            outs.append(_ozaki(a, b))
        finally:
            P.set_ozaki_kernel("auto")
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    with pytest.raises(ValueError):
        P.set_ozaki_kernel("quad")


def _cases(rng, n):
    g = rng.standard_normal((2 * n, n))
    spd = g.T @ g / (2 * n) + 1e-3 * np.eye(n)
    f = np.eye(n) - spd / np.abs(spd).sum(1).max()
    return {
        "gauss": (rng.standard_normal((n, n)), rng.standard_normal((n, n))),
        "wide_rows": (rng.standard_normal((n, n)) * np.exp2(rng.integers(-40, 40, (n, 1))),
                      rng.standard_normal((n, n)) * np.exp2(rng.integers(-40, 40, (1, n)))),
        "wide_entries": (rng.standard_normal((n, n)) * np.exp2(rng.integers(-25, 25, (n, n))),
                         rng.standard_normal((n, n)) * np.exp2(rng.integers(-25, 25, (n, n)))),
        "residual": (f, f),
        "rect": (rng.standard_normal((n, n // 2 + 3)), rng.standard_normal((n // 2 + 3, n + 40))),
    }


@pytest.mark.parametrize("nmod", [16, 14])
def test_emulated_product_bound_and_accuracy(nmod):
    rng = np.random.default_rng(11)
    for name, (a_np, b_np) in _cases(rng, 520).items():
        a, b = torch.from_numpy(a_np).cuda(), torch.from_numpy(b_np).cuda()
        c = _ozaki(a, b, nmod).cpu().numpy()
        ref = a_np.astype(np.longdouble) @ b_np.astype(np.longdouble)
        err = np.abs(c - ref).astype(np.float64)
        pa, pb = _pa_pb(a_np.shape[1], nmod)
        amax = np.abs(a_np).max(1, keepdims=True)
        bmax = np.abs(b_np).max(0, keepdims=True)
        bound = (2.0 ** -pa * amax * np.abs(b_np).sum(0, keepdims=True)
                 + 2.0 ** -pb * bmax * np.abs(a_np).sum(1, keepdims=True)
                 + 2.0 ** -(pa + pb) * a_np.shape[1] * amax * bmax)
        bound = 1.01 * bound + 4 * 2.0 ** -53 * np.abs(ref).astype(np.float64)
        assert np.all(err <= bound), (name, float((err / bound).max()))
        if nmod == 16:
            d = _dmma(a, b).cpu().numpy()
            e_oz = float(np.linalg.norm(err) / np.linalg.norm(ref.astype(np.float64)))
            e_dm = float(np.linalg.norm((d - ref).astype(np.float64)) /
                         np.linalg.norm(ref.astype(np.float64)))
            assert e_oz <= e_dm, (name, e_oz, e_dm)


def test_epilogue_in_place_and_offset_diagonal():
    """D = -A B + C + 2 I (diag shifted by doff), D aliasing C, through si_gemm_ex."""
    import ctypes

    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib

    rng = np.random.default_rng(3)
    m, k, n, doff = 384, 640, 512, 100
    a_np, b_np, c_np = (rng.standard_normal(s) for s in ((m, k), (k, n), (m, n)))
    a, b = torch.from_numpy(a_np).cuda(), torch.from_numpy(b_np).cuda()
    d = torch.from_numpy(c_np).cuda()
    ctr = (ctypes.c_int64 * 2)()
    P.set_gemm_backend("ozaki", 16, 128)
    _lib.call("si_gemm_ex", _lib.handle(), m, n, k, -1.0, a.data_ptr(), k, b.data_ptr(), n, 1.0,
              d.data_ptr(), n, 2.0, doff, d.data_ptr(), n, 0, ctr, _lib.stream_ptr())
    ref = -(a_np.astype(np.longdouble) @ b_np) + c_np
    idx = np.arange(m)
    ref[idx, idx + doff] += 2.0
    out = d.cpu().numpy()
    assert np.abs(out - ref).max() <= 1e-13 * np.abs(ref).max()
    assert ctr[0] == 1


def test_non_finite_zero_and_extreme_rows():
    rng = np.random.default_rng(5)
    n = 300
    a_np = rng.standard_normal((n, n))
    b_np = rng.standard_normal((n, n))
    a_np[3, 7] = np.nan
    a_np[5, 0] = np.inf
    a_np[9] = 0.0
    a_np[11] *= 1e-300
    a_np[13] *= 1e300
    b_np[:, 17] = 0.0
    b_np[4, 21] = -np.inf
    c = _ozaki(torch.from_numpy(a_np).cuda(), torch.from_numpy(b_np).cuda()).cpu().numpy()
    assert np.isnan(c[3]).all() and np.isnan(c[5]).all() and np.isnan(c[:, 21]).all()
    ok_rows = np.setdiff1d(np.arange(n), [3, 5])
    ok_cols = np.setdiff1d(np.arange(n), [21])
    sub = c[np.ix_(ok_rows, ok_cols)]
    assert np.isfinite(sub).all()
    assert (c[9, ok_cols] == 0).all() and (c[ok_rows, 17] == 0).all()
    for i in (11, 13):
        ref = a_np[i].astype(np.longdouble) @ b_np[:, ok_cols]
        assert np.abs(c[i, ok_cols] - ref).max() <= 1e-14 * np.abs(ref).max()


def test_row_split_bitwise_and_deterministic():
    """Rows of the product do not depend on which other rows are computed (the
    block-row sharded path's invariant) nor on the call."""
    rng = np.random.default_rng(9)
    a_np, b_np = rng.standard_normal((1536, 1024)), rng.standard_normal((1024, 1280))
    a, b = torch.from_numpy(a_np).cuda(), torch.from_numpy(b_np).cuda()
    full = _ozaki(a, b)
    assert torch.equal(full, _ozaki(a, b))
    for r0, r1 in ((0, 512), (512, 1100), (1100, 1536)):
        assert torch.equal(_ozaki(a[r0:r1].contiguous(), b), full[r0:r1])


def test_backend_selection():
    import paper_2008_11480_b200 as P

    P.set_gemm_backend("ozaki", 15, 2048)
    assert P.get_gemm_backend() == ("ozaki", 15, 2048)
    rng = np.random.default_rng(1)
    a = torch.from_numpy(rng.standard_normal((1024, 1024))).cuda()
    small = P.mat_mul(a, a, P.MulCounter())  # below min_dim: DMMA, bitwise
    assert torch.equal(small, _dmma(a, a))
    P.set_gemm_backend("ozaki", 15, 2048)
    with pytest.raises(ValueError):
        P.set_gemm_backend("ozaki", 17)
    with pytest.raises(ValueError):
        P.set_gemm_backend("fp32")
    with P.gemm_backend("dmma"):
        assert P.get_gemm_backend()[0] == "dmma"
    assert P.get_gemm_backend() == ("ozaki", 15, 2048)


def _kappa_tol(a, tol=1e-10):
    ev = np.linalg.eigvalsh(a)
    return tol * max(1.0, float(ev.max() / ev.min()) / 1e4)


def test_c3_recipe_emulated_vs_oracle():
    """Config 3 recipe at n=2048 (h8 plan + plain Richardson, 25 iterations) with
    every product emulated: P_k, theta_k within the tolerance at every iteration."""
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    a, b = configs.c3_gram(n=2048)
    tol = _kappa_tol(a)
    P.set_gemm_backend("ozaki", 16, 1024)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    st = P.initial_series(sp, 0, 1, order=8)
    bd = P.as_device(b)
    theta = torch.zeros_like(bd)
    osp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    ost = O.initial_series(osp, 0, 1, 8)
    oth = np.zeros_like(b)
    plan, oplan = P.table_plans()[8][0], O.TABLE_ROOTS[8][0][1]
    for k in range(25):
        theta = P.plain_richardson(theta, st.estimate, sp.matrix, bd, st.ctr)
        st = P.ns_step(st, sp.matrix, plan=plan)
        oth = O.plain_richardson(oth, ost.estimate, osp.matrix, b, ost.ctr)
        ost = O.ns_step(ost, osp.matrix, oplan)
        ep = np.linalg.norm(st.estimate.cpu().numpy() - ost.estimate) / np.linalg.norm(ost.estimate)
        et = np.linalg.norm(theta.cpu().numpy() - oth) / np.linalg.norm(oth)
        assert ep <= tol and et <= tol, (k, ep, et)
    assert (st.ctr.mmm, st.ctr.mvm) == (ost.ctr.mmm, ost.ctr.mvm)


def test_c4_recipe_emulated_vs_oracle():
    """Config 4 recipe (composite rates (2,3,4,5), order_n=2, plain Richardson,
    kappa 1e6) at n=2048, 8 iterations, every product emulated."""
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    a, b = configs.c4_householder(n=2048, rhs=64)
    tol = _kappa_tol(a)
    P.set_gemm_backend("ozaki", 16, 1024)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    st = P.initial_series(sp, 0, 1, order=2)
    bd = P.as_device(b)
    theta = torch.zeros_like(bd)
    osp = O.split_scalar(a, O.inf_norm(a) / 2.0)
    ost = O.initial_series(osp, 0, 1, 2)
    oth = np.zeros_like(b)
    spec = P.CompositeSpec((2, 3, 4, 5))
    for k in range(8):
        theta = P.plain_richardson(theta, st.estimate, sp.matrix, bd, st.ctr)
        st = P.composite_step(st, sp.matrix, sp, spec, 2)
        oth = O.plain_richardson(oth, ost.estimate, osp.matrix, b, ost.ctr)
        ost = O.composite_step(ost, osp.matrix, osp, (2, 3, 4, 5), 2)
        ep = np.linalg.norm(st.estimate.cpu().numpy() - ost.estimate) / np.linalg.norm(ost.estimate)
        et = np.linalg.norm(theta.cpu().numpy() - oth) / np.linalg.norm(oth)
        assert ep <= tol and et <= tol, (k, ep, et)
    assert (st.ctr.mmm, st.ctr.mvm) == (ost.ctr.mmm, ost.ctr.mvm)


def test_chunks_bitwise():
    """Chunking D (bounded workspace, si_set_ozaki_chunks) changes nothing: every
    row's and column's scale and residues are its own; the epilogue's C and the
    shifted diagonal follow the chunk offsets; B-side planes are rebuilt per row
    chunk when several column chunks are needed."""
    import ctypes

    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib

    rng = np.random.default_rng(21)
    m, k, n, doff = 1300, 1100, 1300, 37
    a_np, b_np, c_np = (rng.standard_normal(s) for s in ((m, k), (k, n), (m, n)))
    a, b, c = (torch.from_numpy(x).cuda() for x in (a_np, b_np, c_np))
    P.set_gemm_backend("ozaki", 16, 128)
    outs = []
    try:
        for rows, cols in ((0, 0), (0, 256), (0, 768), (512, 0), (256, 512), (768, 256)):
            P.set_ozaki_chunks(rows, cols)
            d = torch.empty(m, n, dtype=torch.float64, device="cuda")
            ctr = (ctypes.c_int64 * 2)()
            _lib.call("si_gemm_ex", _lib.handle(), m, n, k, -1.0, a.data_ptr(), k, b.data_ptr(), n,
                      1.0, c.data_ptr(), n, 3.0, doff, d.data_ptr(), n, 0, ctr, _lib.stream_ptr())
            outs.append(d)
    finally:
        P.set_ozaki_chunks(0, 0)
    for d in outs[1:]:
        assert torch.equal(d, outs[0])
    ref = -(a_np.astype(np.longdouble) @ b_np) + c_np
    idx = np.arange(m - doff)
    ref[idx, idx + doff] += 3.0
    assert np.abs(outs[0].cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()
    with pytest.raises(ValueError):
        P.set_ozaki_chunks(-1, 0)


def test_workspace_retry_under_memory_cap():
    """With the allocator capped below a product's full workspace (3 x 1 GiB of
    residue / result planes at n=8192), the library retries with smaller row x
    column chunks instead of failing, and the result is bitwise the uncapped one."""
    import paper_2008_11480_b200 as P

    n = 8192
    g = torch.Generator(device="cuda").manual_seed(4)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    full = _ozaki(a, b)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    total = torch.cuda.get_device_properties(0).total_memory
    used = torch.cuda.memory_allocated()
    # room for the output (0.5 GiB) and ~1.5 GiB of workspace, not the 3.2 GiB of one chunk
    torch.cuda.set_per_process_memory_fraction((used + (2 << 30)) / total)
    try:
        capped = _ozaki(a, b)
        torch.cuda.synchronize()
    finally:
        torch.cuda.set_per_process_memory_fraction(1.0)
        torch.cuda.empty_cache()
    assert torch.equal(capped, full)


def test_step_operand_images_kept_bitwise():
    """A composite step keeps the scales / residue planes of its immutable
    inputs (A, S^-1, B, G, F) across its emulated products; the parts on
    concurrent streams recompute them per product.  Both give the same bits,
    and the kept images save residue launches."""
    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib, configs

    a, _ = configs.c4_householder(n=2048, rhs=1)
    P.set_gemm_backend("ozaki", 16, 1024)
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False)
    st = P.initial_series(sp, 0, 1, order=2)
    spec = P.CompositeSpec((2, 3, 4, 5))
    h = _lib.handle()
    import ctypes

    def run(executor):
        _lib.call("si_profile_begin", h)
        out = P.composite_step(st, sp.matrix, sp, spec, 2, executor=executor)
        torch.cuda.synchronize()
        ms, fl, ng, nl = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        _lib.call("si_profile_end", h, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(ng),
                  ctypes.byref(nl))
        return out, nl.value

    serial, n_serial = run(None)
    conc, n_conc = run("streams")
    assert torch.equal(serial.estimate, conc.estimate)
    assert torch.equal(serial.residual, conc.residual)
    assert serial.ctr.mmm == conc.ctr.mmm
    assert n_serial < n_conc, (n_serial, n_conc)


def test_strided_operands_through_the_abi():
    """Operands and outputs with leading dimensions larger than their widths
    (sub-blocks of bigger buffers), odd K: the emulated si_gemm_ex equals the
    same product on contiguous copies, bitwise, and meets the accuracy bound."""
    import ctypes

    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib

    rng = np.random.default_rng(41)
    m, k, n = 700, 1031, 900
    big_a = torch.from_numpy(rng.standard_normal((m, k + 77))).cuda()
    big_b = torch.from_numpy(rng.standard_normal((k, n + 33))).cuda()
    big_c = torch.from_numpy(rng.standard_normal((m, n + 5))).cuda()
    a, b, c = big_a[:, 3:3 + k], big_b[:, :n], big_c[:, 2:2 + n]
    P.set_gemm_backend("ozaki", 16, 128)
    ctr = (ctypes.c_int64 * 2)()
    big_d = torch.full((m, n + 11), 7.0, dtype=torch.float64, device="cuda")
    d = big_d[:, 4:4 + n]
    _lib.call("si_gemm_ex", _lib.handle(), m, n, k, 1.0, a.data_ptr(), a.stride(0), b.data_ptr(),
              b.stride(0), 1.0, c.data_ptr(), c.stride(0), 0.0, 0, d.data_ptr(), d.stride(0), 0,
              ctr, _lib.stream_ptr())
    ac, bc, cc = a.contiguous(), b.contiguous(), c.contiguous()
    dc = torch.empty(m, n, dtype=torch.float64, device="cuda")
    _lib.call("si_gemm_ex", _lib.handle(), m, n, k, 1.0, ac.data_ptr(), k, bc.data_ptr(), n, 1.0,
              cc.data_ptr(), n, 0.0, 0, dc.data_ptr(), n, 0, ctr, _lib.stream_ptr())
    assert torch.equal(d, dc)
    assert bool((big_d[:, :4] == 7.0).all()) and bool((big_d[:, 4 + n:] == 7.0).all())
    ref = a.cpu().numpy().astype(np.longdouble) @ b.cpu().numpy() + c.cpu().numpy()
    assert np.abs(d.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()


def test_largest_inner_dimension():
    """K = 65536 (kMaxK): all -128 residues give the largest int32 sum the
    epilogue reduces, 2^30 (u = 2^31), exactly; an emulated product with that K
    meets the a-priori bound."""
    import paper_2008_11480_b200 as P

    kp = 65536
    mods = P.ozaki_moduli(2)
    a = torch.full((2, 128, kp), -128, dtype=torch.int8, device="cuda")
    bt = torch.full((2, 128, kp), -128, dtype=torch.int8, device="cuda")
    for kernel in ("single", "pair"):
        P.set_ozaki_kernel(kernel)
        try:
            r = P.i8_gemm_mod(a, bt)
        finally:
            P.set_ozaki_kernel("auto")
        for l in range(2):
            assert bool((r[l] == (kp * 16384) % mods[l]).all()), (kernel, l)
    rng = np.random.default_rng(13)
    a_np, b_np = rng.standard_normal((256, kp)), rng.standard_normal((kp, 256))
    c = _ozaki(torch.from_numpy(a_np).cuda(), torch.from_numpy(b_np).cuda()).cpu().numpy()
    ref = a_np.astype(np.longdouble) @ b_np.astype(np.longdouble)
    pa, pb = _pa_pb(kp, 16)
    amax = np.abs(a_np).max(1, keepdims=True)
    bmax = np.abs(b_np).max(0, keepdims=True)
    bound = (2.0 ** -pa * amax * np.abs(b_np).sum(0, keepdims=True)
             + 2.0 ** -pb * bmax * np.abs(a_np).sum(1, keepdims=True)
             + 2.0 ** -(pa + pb) * kp * amax * bmax)
    bound = 1.01 * bound + 4 * 2.0 ** -53 * np.abs(ref).astype(np.float64)
    assert np.all(np.abs(c - ref).astype(np.float64) <= bound)
