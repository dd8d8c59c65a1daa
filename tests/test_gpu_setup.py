"""Setup path on the device against the reference's
outputs (tests/golden/setup.npz, made by the unmodified reference) and, at
config-4 size, against the oracle:

* the fused symmetry check + symmetrize pass (splitting.py:67-73),
* the blocked Cholesky positive-definiteness check with the reference's pivot
  floor (splitting.py:76-98), including exactly singular pivots,
* the device power iteration (matrix_core.py:183-239).
"""

import ctypes
import time

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


def test_symmetrize_checked_matches_reference():
    from paper_2008_11480_b200.splitting import _symmetrized

    g = golden("setup.npz")
    for i in range(5):
        a = g[f"sym{i}_a"]
        if int(g[f"sym{i}_ok"]):
            out = _symmetrized(a).cpu().numpy()
            assert np.array_equal(out, g[f"sym{i}_out"])  # (a + a.T) / 2.0, bitwise
        else:
            with pytest.raises(ValueError, match="symmetric"):
                _symmetrized(a)
    bad = np.eye(40)
    bad[3, 17] = np.nan
    with pytest.raises(ValueError, match="finite"):
        _symmetrized(bad)


@pytest.mark.parametrize("n", [1, 31, 33, 1000, 4099])
def test_symmetrize_checked_norms_and_in_place(n):
    from paper_2008_11480_b200 import _lib

    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    t = torch.as_tensor(a, device="cuda")
    ref_out = (a + a.T) / 2.0
    vals = [ctypes.c_double() for _ in range(3)]
    h, s = _lib.handle(0), _lib.stream_ptr()
    _lib.call("si_symmetrize_checked", h, n, t.data_ptr(), t.data_ptr(), *map(ctypes.byref, vals), s)
    asym, fro, bad = (v.value for v in vals)
    assert np.array_equal(t.cpu().numpy(), ref_out)  # in place
    assert bad == 0.0
    assert asym == pytest.approx(np.linalg.norm(a - a.T), rel=1e-12, abs=1e-300)
    assert fro == pytest.approx(np.linalg.norm(a), rel=1e-12)


def test_symmetrize_checked_full_size():
    """n=16384: one pass, no n^2 temporaries; symmetric input accepted and
    returned bitwise, a 1e-8 relative asymmetry rejected."""
    from paper_2008_11480_b200 import configs
    from paper_2008_11480_b200.splitting import _symmetrized

    a, _ = configs.c4_householder_device(n=16384, rhs=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = _symmetrized(a)
    dt = time.perf_counter() - t0
    assert torch.equal(out, a)  # a is exactly symmetric: (a + a^T)/2 == a
    print(f"symmetrize_checked n=16384: {dt * 1e3:.2f} ms incl. host read-back "
          f"({2 * 8 * 16384**2 / dt / 1e9:.0f} GB/s)")
    del out
    a[5, 7] += 1e-8 * float(torch.linalg.norm(a))
    with pytest.raises(ValueError, match="symmetric"):
        _symmetrized(a)


def test_pd_verdicts_match_reference():
    import paper_2008_11480_b200 as P

    g = golden("setup.npz")
    for i in range(int(g["pd_count"])):
        a = g[f"pd{i}_a"]
        assert int(P.is_positive_definite(a)) == int(g[f"pd{i}_default"]), i
        assert int(P.is_positive_definite(a, pivot_tol=0.0)) == int(g[f"pd{i}_zero_tol"]), i


def _pd_info(a, pivot_tol=None):
    from paper_2008_11480_b200 import _lib

    is_pd, idx, piv = ctypes.c_int(), ctypes.c_int64(), ctypes.c_double()
    _lib.call("si_is_positive_definite", _lib.handle(0), a.shape[0], a.data_ptr(), a.shape[0],
              0.0 if pivot_tol is None else pivot_tol, 1 if pivot_tol is None else 0,
              ctypes.byref(is_pd), ctypes.byref(idx), ctypes.byref(piv), _lib.stream_ptr())
    return bool(is_pd.value), idx.value, piv.value


@pytest.mark.parametrize("n", [4096, 16384])
def test_pd_verdicts_at_size_vs_oracle(n):
    """Config 4's matrix (kappa 1e6, spectrum known exactly: lambda in [1, 1e6]):
    SPD -> PD; shifted by -2 I (smallest eigenvalue min(lambda) - 2 < 0) -> not
    PD; a block-diagonal matrix with an exactly singular 2x2 block
    [[1, 1], [1, 1 + 1e-16]] at rows m, m+1 -> not PD at pivot m+1 (early exit).
    Against the oracle's blocked restatement of splitting.py:76-98: every
    verdict at n=4096; at n=16384 the SPD verdict (the other two follow from
    the known spectrum / the exact block, and cost minutes of host time)."""
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    a, _ = configs.c4_householder_device(n=n, rhs=1)
    lam, _, _ = configs._c4_draws(n, 64, 1, 0)
    assert lam.min() > 1e-12 * n * lam.max()  # far above the pivot floor
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ok, idx, _ = _pd_info(a)
    dt = time.perf_counter() - t0
    print(f"is_positive_definite n={n}: {dt * 1e3:.1f} ms ({n**3 / 3 / dt / 1e12:.1f} "
          f"TFLOP/s of n^3/3)")
    assert ok and idx == -1
    assert O.is_positive_definite_blocked(a.cpu().numpy(), nb=1024)
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    a -= 2.0 * eye
    ok2, _, piv2 = _pd_info(a)
    assert lam.min() - 2.0 < 0
    assert not ok2 and piv2 <= 1e-12 * float(torch.max(torch.sum(torch.abs(a), dim=1)))
    if n <= 4096:
        assert not O.is_positive_definite_blocked(a.cpu().numpy(), nb=1024)
    a += 2.0 * eye
    del eye
    m = n // 2 - 192  # inside a 128-row panel, not at its start
    a[m:m + 2, :] = 0.0
    a[:, m:m + 2] = 0.0
    a[m:m + 2, m:m + 2] = torch.tensor([[1.0, 1.0], [1.0, 1.0 + 1e-16]], dtype=torch.float64)
    t0 = time.perf_counter()
    ok3, idx3, piv3 = _pd_info(a)
    dt3 = time.perf_counter() - t0
    assert not ok3 and idx3 == m + 1 and piv3 == 0.0
    if n <= 4096:
        assert not O.is_positive_definite_blocked(a.cpu().numpy(), nb=1024)
    print(f"singular pivot at {m + 1} found in {dt3 * 1e3:.1f} ms (early exit)")


def test_spectral_radius_matches_reference():
    import paper_2008_11480_b200 as P

    g = golden("setup.npz")
    for i in range(int(g["rho_count"])):
        got = P.spectral_radius(g[f"rho{i}_a"])
        want = float(g[f"rho{i}"])
        assert got == pytest.approx(want, rel=1e-10, abs=0.0), i
    # a rotation times a scaling: |est| oscillates and never settles
    rot = np.array([[np.cos(1.0), -np.sin(1.0)], [np.sin(1.0), np.cos(1.0)]]) @ np.diag([1.0, 0.5])
    with pytest.raises(P.SpectralRadiusError):  # the oracle (and the reference) raise too
        P.spectral_radius(rot, max_iter=300)


def test_spectral_radius_large_known_spectrum():
    """n=2048, spectrum {0.95} U [-0.5, 0.5]: the device loop (host checks every
    32 iterations) reaches the oracle's estimate."""
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as O

    n = 2048
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = rng.uniform(-0.5, 0.5, n)
    ev[0] = 0.95
    m = (q * ev) @ q.T
    t0 = time.perf_counter()
    got = P.spectral_radius(m)
    dt = time.perf_counter() - t0
    want = O.spectral_radius(m)
    assert got == pytest.approx(want, rel=1e-11)
    assert got == pytest.approx(0.95, rel=1e-10)
    print(f"spectral_radius n={n}: {got!r} in {dt * 1e3:.1f} ms (oracle {want!r})")
