"""The C-ABI library: loads without a GPU and exports every symbol the header declares."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "seriesinv_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SI_API\s+(?:const\s+)?\w+\*?\s+(si_\w+)\s*\(", text)))


def test_header_declares_the_step_seam():
    syms = declared_symbols()
    for name in ("si_gemm", "si_ns_step", "si_composite_step", "si_double_ns_step",
                 "si_richardson_step", "si_richardson_recursive_step", "si_plain_richardson",
                 "si_batched_composite_richardson", "si_nested_eval", "si_geometric_apply"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2008_11480_b200 import _lib

    lib = _lib.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.si_version() == 1


def test_python_prototypes_cover_the_header():
    from paper_2008_11480_b200 import _lib

    declared = set(declared_symbols()) - {"si_version", "si_last_error"}
    assert declared == set(_lib.SIGNATURES)


def test_prototype_arity_matches_header():
    from paper_2008_11480_b200 import _lib

    text = open(HEADER).read()
    for name, argtypes in _lib.SIGNATURES.items():
        m = re.search(rf"{name}\s*\(([^;]*)\);", text, re.S)
        assert m, name
        body = re.sub(r"\(\*(\w+)\)\s*\([^()]*\)", r"(*\1)", m.group(1))  # fn-pointer params
        params = [p for p in body.split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(argtypes), name


def test_no_silent_cpu_fallback():
    """Without a CUDA device the product path raises instead of computing on the host."""
    import torch

    import paper_2008_11480_b200 as P
    from paper_2008_11480_b200 import _lib

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(_lib.NativeUnavailable):
        P.mat_mul([[1.0]], [[1.0]], P.MulCounter())
    with pytest.raises(_lib.NativeUnavailable):
        _lib.handle()


def test_abi_rejects_bad_arguments_without_gpu():
    """Argument validation happens before any device work and maps to SI_EINVAL."""
    from paper_2008_11480_b200 import _lib

    lib = _lib.load_library()
    assert lib.si_create(0, None) == _lib.SI_EINVAL
    assert b"null" in lib.si_last_error()
    buf = ctypes.c_void_p()
    assert lib.si_gemm(None, 1, 1, 1, 1.0, None, 1, None, 1, 0.0, None, 1, 0.0, None, 1, 0, None,
                       None) == _lib.SI_EINVAL
    del buf


def test_baked_resident_programs_are_current():
    """The compile-time programs of the config-1/2 resident kernels
    (csrc/resident_fixed_c*.inc, tools/gen_resident_fixed.py) equal what the
    library's recorder / scheduler / allocator build today (host-only entry
    points, no device): a stale file would silently fall back to the
    interpreter."""
    import ctypes
    import os

    from paper_2008_11480_b200 import _lib
    from paper_2008_11480_b200.series_toolkit import encode_many, geometric_base_plan

    lib = _lib.load_library()
    csrc = os.path.join(os.path.dirname(_lib.__file__), "csrc")

    def body(path):
        with open(path) as fh:
            return "".join(ln for ln in fh if not ln.startswith("//"))

    code, offsets, consts = encode_many([geometric_base_plan(x) for x in (2, 3)])
    n = ctypes.c_int64()
    args = [32, 2, _lib.i32_array([2, 3]), _lib.i32_array(code), _lib.i64_array(offsets),
            _lib.f64_array(consts), len(consts), 2]
    assert lib.si_resident_program_source(*args, None, 0, ctypes.byref(n)) == 0
    buf = ctypes.create_string_buffer(n.value + 1)
    assert lib.si_resident_program_source(*args, buf, n.value + 1, ctypes.byref(n)) == 0
    assert buf.value.decode() == body(os.path.join(csrc, "resident_fixed_c2.inc"))
    assert lib.si_resident_program_source_ns(64, 3, 8, None, 0, ctypes.byref(n)) == 0
    buf = ctypes.create_string_buffer(n.value + 1)
    assert lib.si_resident_program_source_ns(64, 3, 8, buf, n.value + 1, ctypes.byref(n)) == 0
    assert buf.value.decode() == body(os.path.join(csrc, "resident_fixed_c1.inc"))


def test_backend_entry_points_validate_without_gpu():
    """The FP64-product backend entry points (si_set_gemm_backend & co.) reject
    bad arguments with SI_EINVAL before touching a device."""
    from paper_2008_11480_b200 import _lib

    lib = _lib.load_library()
    E = _lib.SI_EINVAL
    assert lib.si_set_gemm_backend(None, 1, 16, 1024) == E  # null handle
    assert lib.si_get_gemm_backend(None, None, None, None) == E
    assert lib.si_set_ozaki_chunks(None, 0, 0) == E
    assert lib.si_set_ozaki_kernel(None, 0) == E
    assert lib.si_ozaki_tune(-1, 0, 0) == E
    assert lib.si_ozaki_tune(0, 3, 0) == E
    assert lib.si_ozaki_tune_stages(2) == E and lib.si_ozaki_tune_stages(7) == E
    assert lib.si_ozaki_tune_ksplit(-128) == E and lib.si_ozaki_tune_ksplit(100) == E
    assert lib.si_ozaki_moduli(0, None) == E
    mods = (ctypes.c_uint32 * 17)()
    assert lib.si_ozaki_moduli(17, mods) == E
    assert lib.si_ozaki_moduli(16, mods) == _lib.SI_OK
    assert list(mods)[:3] == [256, 255, 253]
    assert lib.si_i8_gemm_mod(None, None, None, None, 1, 1, 128, 1, None) == E
    assert lib.si_profile_i8(None, None, None, None) == E


def test_step_norm_entry_point_validates_without_gpu():
    """si_set_step_norm (the fused ||F'||_F^2 target of the next step call)
    rejects a null handle; a step call with a null handle still returns
    SI_EINVAL (it consumes a target before its argument checks)."""
    from paper_2008_11480_b200 import _lib

    lib = _lib.load_library()
    assert lib.si_set_step_norm(None, None) == _lib.SI_EINVAL
    assert lib.si_ns_step(None, 4, None, None, None, 2, None, 0, None, 0, None, None, None,
                          None) == _lib.SI_EINVAL
