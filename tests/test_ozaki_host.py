"""Host-side checks of the Ozaki-II emulation's integer arithmetic (csrc/ozaki.cu),
restated with exact Python / numpy integers -- no GPU needed:

* the moduli the library reports are pairwise coprime, <= 256, and their
  product M is large enough for the scaling rule K 2^(pa+pb) <= M / 4 with
  pa, pb >= 53 at K <= 32768 (16 moduli),
* the int32 accumulator bound |C_l| <= K 2^14 < 2^30 + 1 for every K <= kMaxK,
* the epilogue's magic-multiply reduction q = floor(u * magic / 2^39) is the
  exact quotient u // m for every u in [0, 2^31] (checked on every u = -1 mod m,
  the worst case, and on the boundaries),
* the residue kernels' chunked reduction (u = c2 2^40 + c1 2^20 + c0 with the
  2^57 offset, shifted by m / 2) gives the symmetric residue of the integer
  image, and the byte packing's carry-free per-byte subtraction equals the
  int8 two's-complement of r - h.
"""

import math

import numpy as np
import pytest

K_MAX = 65536


def _moduli():
    from paper_2008_11480_b200 import _lib

    try:
        _lib.load_library()
    except Exception as exc:  # noqa: BLE001 -- library not built here
        pytest.skip(f"library not loadable: {exc}")
    import ctypes

    out = (ctypes.c_uint32 * 16)()
    _lib.call("si_ozaki_moduli", 16, out)
    return [int(x) for x in out]


def _pa_pb(k, nmod, mods):
    m = math.prod(mods[:nmod])
    bits = m.bit_length() - 1  # 2^bits <= M
    lk = max(0, (k - 1).bit_length())
    t = bits - 2 - lk
    return min(56, (t + 1) // 2), min(56, t // 2), m


def test_moduli_and_scaling_rule():
    mods = _moduli()
    assert len(set(mods)) == 16 and all(2 <= m <= 256 for m in mods)
    for i in range(16):
        for j in range(i + 1, 16):
            assert math.gcd(mods[i], mods[j]) == 1
    for nmod in range(8, 17):
        for k in (1, 2, 127, 128, 1000, 4096, 16384, 32768, K_MAX):
            pa, pb, m = _pa_pb(k, nmod, mods)
            assert k * 2 ** (pa + pb) <= m // 4
    pa, pb, _ = _pa_pb(16384, 16, mods)
    assert (pa, pb) == (55, 54)
    pa, pb, _ = _pa_pb(32768, 16, mods)
    assert min(pa, pb) >= 53


def test_int32_accumulator_bound():
    # symmetric residues lie in [-128, 127]: |a b| <= 2^14 per term
    assert K_MAX * 2 ** 14 <= 2 ** 30


def test_epilogue_magic_reduction_exact():
    mods = _moduli()
    for m in mods:
        magic = (1 << 39) // m + 1
        off = (1 << 30) % m
        # worst case of the magic multiply: u = -1 (mod m), all of [0, 2^31]
        u = np.arange(m - 1, (1 << 31) + 1, m, dtype=np.uint64)
        q = (u * np.uint64(magic)) >> np.uint64(39)
        assert np.array_equal(q, u // np.uint64(m)), m
        for uu in (0, 1, m - 1, m, (1 << 30) - 1, 1 << 30, (1 << 31) - 1, 1 << 31):
            assert (uu * magic) >> 39 == uu // m
        # the stored residue of v = u - 2^30: (u mod m - 2^30 mod m) mod m
        for v in (-(1 << 30), -1, 0, 1, 12345, (1 << 30) - 1, 1 << 30):
            uu = v + (1 << 30)
            r = uu - ((uu * magic) >> 39) * m
            r = r - off if r >= off else r + m - off
            assert r == v % m


def _res_shifted(x, m):
    """csrc/ozaki.cu res_shifted: (x + m/2) mod m from the 20-bit chunks of x + 2^57."""
    u = x + (1 << 57)
    c0, c1, c2 = u & 0xFFFFF, (u >> 20) & 0xFFFFF, u >> 40
    r40, r20 = pow(2, 40, m), pow(2, 20, m)
    kh = (m - pow(2, 57, m) + m // 2) % m
    v = c2 * r40 + c1 * r20 + c0 + kh
    assert v < 2 ** 29
    return v % m


def _sub_bytes(w, h):
    """csrc/ozaki.cu pack_sym4's carry-free per-byte add of (256 - h)."""
    hh = ((256 - h) & 0xFF) * 0x01010101
    return (((w & 0x7F7F7F7F) + (hh & 0x7F7F7F7F)) ^ ((w ^ hh) & 0x80808080)) & 0xFFFFFFFF


def test_residue_chunks_and_packing():
    mods = _moduli()
    rng = np.random.default_rng(0)
    xs = [0, 1, -1, (1 << 56), -(1 << 56), (1 << 55) + 12345, -(1 << 55) - 999]
    xs += [int(v) for v in rng.integers(-(1 << 56), 1 << 56, 200, dtype=np.int64)]
    for m in mods:
        h = m // 2
        for x in xs:
            r = _res_shifted(x, m)
            sym = r - h
            assert -128 <= sym <= 127 and (sym - x) % m == 0
            # the symmetric representative the GEMM bound assumes
            ref = x % m
            ref = ref - m if ref >= (m + 1) // 2 else ref
            assert sym == ref, (m, x)
        rs = [_res_shifted(x, m) for x in xs[:4]]
        w = rs[0] | (rs[1] << 8) | (rs[2] << 16) | (rs[3] << 24)
        got = _sub_bytes(w, h)
        for j in range(4):
            byte = (got >> (8 * j)) & 0xFF
            assert (byte - 256 if byte >= 128 else byte) == rs[j] - h
