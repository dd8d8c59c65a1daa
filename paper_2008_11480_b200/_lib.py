"""ctypes binding of ``libseriesinv_b200.so`` (the C ABI in include/seriesinv_b200.h).

The product path has no fallback: if the shared library is missing or no CUDA
device is visible, every entry point raises.  Device memory and streams come
from PyTorch (plumbing only); all arithmetic runs in the library's kernels.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_void_p

import torch

LIB_NAME = "libseriesinv_b200.so"
LIB_PATH = os.environ.get("SI_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

SI_OK, SI_EINVAL, SI_ECUDA, SI_ENOMEM = 0, -1, -2, -3

_P = c_void_p
_I64 = c_int64
_I = c_int
_D = c_double
_PI64 = POINTER(c_int64)

# name -> argtypes (all return int status)
SIGNATURES: dict[str, list] = {
    "si_create": [_I, POINTER(c_void_p)],
    "si_destroy": [_P],
    "si_trim": [_P],
    "si_set_allocator": [_P, _P, _P, _P],
    "si_gemm": [_P, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64, _D, _P, _I64, _I, _PI64, _P],
    "si_gemm_ex": [_P, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64, _D, _I64, _P, _I64, _I, _PI64, _P],
    "si_gemm_panels": [_P, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64, _D, _I64, _P,
                       _I64, _P, ctypes.c_uint32, _P, _I, _I, _PI64, _P],
    "si_sym_alloc": [_P, ctypes.c_size_t, POINTER(c_void_p), _P],
    "si_sym_free": [_P, _P],
    "si_sym_open": [_P, _P, POINTER(c_void_p)],
    "si_sym_close": [_P, _P],
    "si_stream_write_u32": [_P, _P, ctypes.c_uint32, _P],
    "si_stream_wait_u32": [_P, _P, ctypes.c_uint32, _P],
    "si_copy_async": [_P, _P, _P, ctypes.c_size_t, _P],
    "si_lincomb": [_P, _I64, _I64, _D, _I, _P, _P, _P, _P, _I64, _P],
    "si_lincomb_ex": [_P, _I64, _I64, _D, _I64, _I, _P, _P, _P, _P, _I64, _P],
    "si_fro_norm": [_P, _I64, _I64, _P, _I64, POINTER(c_double), _P],
    "si_set_step_norm": [_P, _P],
    "si_inf_norm": [_P, _I64, _I64, _P, _I64, POINTER(c_double), _P],
    "si_split_scalar": [_P, _I64, _P, _D, _P, _P, _P],
    "si_split_diagonal": [_P, _I64, _P, _P, _P, _P],
    "si_symmetrize": [_P, _I64, _P, _P, _P],
    "si_symmetrize_checked": [_P, _I64, _P, _P, POINTER(c_double), POINTER(c_double),
                              POINTER(c_double), _P],
    "si_is_positive_definite": [_P, _I64, _P, _I64, _D, _I, POINTER(c_int), _PI64,
                                POINTER(c_double), _P],
    "si_resident_program_source": [_I64, _I, _P, _P, _P, _P, _I64, _I, _P, _I64, _PI64],
    "si_resident_program_source_ns": [_I64, _I, _I, _P, _I64, _PI64],
    "si_comm_unique_id": [_P],
    "si_comm_create_nccl": [_P, _I, _I, _P, _I64, POINTER(c_void_p)],
    "si_comm_create_callback": [_I, _I, _I64, _P, _P, _P, POINTER(c_void_p)],
    "si_comm_destroy": [_P],
    "si_comm_rows": [_P, _PI64, _PI64, _PI64, _PI64],
    "si_sharded_ns_step": [_P, _P, _I64, _P, _P, _P, _I, _P, _I64, _P, _I64, _P, _P, _PI64, _P],
    "si_sharded_composite_step": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I64,
                                  _I, _P, _P, _PI64, _P],
    "si_sharded_richardson_recursive_step": [
        _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _I64, _P, _I64, _I,
        _P, _P, _P, _P, _P, _P, _P, _PI64, _P,
    ],
    "si_sharded_plain_richardson": [_P, _P, _I64, _I64, _P, _P, _P, _P, _P, _PI64, _P],
    "si_sharded_fro_norm": [_P, _P, _I64, _I64, _P, POINTER(c_double), _P],
    "si_power_iterate": [_P, _I64, _P, _I64, _P, _D, _I64, _I, POINTER(c_double),
                         POINTER(c_double), _PI64, POINTER(c_int), _P],
    "si_horner_eval": [_P, _I64, _P, _P, _I, _P, _I, _P, _PI64, _P],
    "si_factored_eval": [_P, _I64, _P, _P, _P, _I, _I, _I, _P, _PI64, _P],
    "si_nested_eval": [_P, _I64, _P, _P, _P, _P, _I64, _P, _I64, _I, _P, _PI64, _P],
    "si_geometric_apply": [_P, _I64, _P, _P, _I, _P, _P, _I64, _P, _I64, _P, _PI64, _P],
    "si_mat_pow_counted": [_P, _I64, _P, _I, _P, _PI64, _P],
    "si_initial_series": [_P, _I64, _P, _P, _P, _I, _I, _P, _P, _PI64, _P],
    "si_ns_step": [_P, _I64, _P, _P, _P, _I, _P, _I64, _P, _I64, _P, _P, _PI64, _P],
    "si_ns_step_ex": [_P, _I64, _P, _P, _P, _I, _P, _I64, _P, _I64, _P, _P, _P, _P, _PI64, _P],
    "si_ns_step_gated": [_P, _I64, _P, _P, _P, _I, _P, _I64, _P, _I64, _P, ctypes.c_uint32, _I, _P,
                         _P, _I, _P, _P, _PI64, _P],
    "si_composite_step": [_P, _I64, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I64, _I, _I, _P, _P, _PI64, _P],
    "si_composite_step_ex": [_P, _I64, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I64, _I, _I, _P, _P, _P, _P, _PI64, _P],
    "si_composite_step_gated": [_P, _I64, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I64, _I, _I,
                                _P, ctypes.c_uint32, _I, _P, _P, _I, _P, _P, _PI64, _P],
    "si_composite_parts": [_P, _I64, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I64, _P, _P, _PI64, _P],
    "si_composite_apply": [_P, _I64, _P, _P, _P, _P, _P, _I, _P, _P, _PI64, _P],
    "si_initial_double": [_P, _I64, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _PI64, _P],
    "si_double_ns_step": [_P, _I64, _P, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _PI64, _P],
    "si_additive_correction_step": [_P, _I64, _P, _P, _P, _I, _P, _P, _PI64, _P],
    "si_richardson_step": [_P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _PI64, _P],
    "si_richardson_recursive_step": [
        _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _I64, _P, _I64, _I, _I,
        _P, _P, _P, _P, _P, _P, _P, _PI64, _P,
    ],
    "si_richardson_recursive_step_ex": [
        _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _I64, _P, _I64, _I, _I,
        _P, _P, _P, _P, _P, _P, _P, _P, _P, _PI64, _P,
    ],
    "si_plain_richardson": [_P, _I64, _I64, _P, _P, _P, _P, _P, _PI64, _P],
    "si_profile_begin": [_P],
    "si_profile_end": [_P, POINTER(c_double), POINTER(c_double), _PI64, _PI64],
    "si_dmma_peak": [_P, _I, POINTER(c_double)],
    "si_set_gemm_backend": [_P, _I, _I, _I64],
    "si_get_gemm_backend": [_P, POINTER(c_int), POINTER(c_int), _PI64],
    "si_ozaki_moduli": [_I, POINTER(ctypes.c_uint32)],
    "si_set_ozaki_chunks": [_P, _I64, _I64],
    "si_set_ozaki_kernel": [_P, _I],
    "si_ozaki_tune": [_I, _I, _I],
    "si_ozaki_tune_stages": [_I],
    "si_ozaki_tune_ksplit": [_I64],
    "si_i8_gemm_mod": [_P, _P, _P, _P, _I64, _I64, _I64, _I, _P],
    "si_profile_i8": [_P, POINTER(c_double), POINTER(c_double), _PI64],
    "si_batched_ns_richardson": [_P, _I64, _I64, _P, _P, _I, _P, _I64, _P, _I64, _I, _P, _P, _P, _PI64, _P],
    "si_batched_composite_richardson": [
        _P, _I64, _I64, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I64, _I, _I, _P, _P, _P, _PI64, _P,
    ],
    "si_batched_ns_richardson_ex": [_P, _I64, _I64, _P, _P, _I, _P, _I64, _P, _I64, _I, _P, _P, _P,
                                    _P, _P, _P, _PI64, _P],
    "si_batched_composite_richardson_ex": [
        _P, _I64, _I64, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I64, _I, _I, _P, _P, _P, _P, _P, _P,
        _PI64, _P,
    ],
    "si_batched_composite_richardson_gated": [
        _P, _I64, _I64, _P, _P, _P, _P, _I, _P, _P, _P, _P, _I64, _I, _I, _P, _P, _P, _P, _P, _P,
        _P, ctypes.c_uint32, _I64, _P, _PI64, _P,
    ],
}

_lib = None
_lib_lock = threading.Lock()
_handles: dict[int, int] = {}


class NativeUnavailable(RuntimeError):
    """The CUDA extension is not built or no CUDA device is visible."""


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every prototype (no GPU needed)."""
    global _lib
    if _lib is not None and path == LIB_PATH:  # loaded: no lock on the hot path
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(path)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = c_int
        lib.si_last_error.restype = ctypes.c_char_p
        lib.si_last_error.argtypes = []
        lib.si_version.restype = c_int
        lib.si_version.argtypes = []
        _lib = lib
        return lib


def _raise(status: int, name: str):
    msg = _lib.si_last_error().decode(errors="replace") if _lib is not None else ""
    if status == SI_EINVAL:
        raise ValueError(msg or f"{name}: invalid argument")
    if status == SI_ENOMEM:
        raise MemoryError(f"{name}: {msg}")
    raise RuntimeError(f"{name} failed ({status}): {msg}")


_ALLOC_FN = ctypes.CFUNCTYPE(c_void_p, c_void_p, ctypes.c_size_t, c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, c_void_p, c_void_p, c_void_p)


def _torch_alloc(ctx, nbytes, stream):
    try:
        return torch.cuda.caching_allocator_alloc(int(nbytes), device=int(ctx or 0),
                                                  stream=int(stream or 0))
    except Exception:  # noqa: BLE001 -- reported to C as NULL (SI_ENOMEM)
        return None


def _torch_free(ctx, ptr, stream):
    torch.cuda.caching_allocator_delete(int(ptr))


# kept alive for the lifetime of the process (C holds the raw pointers)
_ALLOC_CB = _ALLOC_FN(_torch_alloc)
_FREE_CB = _FREE_FN(_torch_free)


def handle(device: int | None = None) -> int:
    """Per-device library handle (side streams, events); the library's
    temporaries are allocated from PyTorch's caching allocator so one allocator
    owns all device memory."""
    if _handles:  # fast path: a handle exists, so CUDA and the library are up
        h = _handles.get(torch.cuda.current_device() if device is None else int(device))
        if h is not None:
            return h
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the seriesinv B200 path has no CPU fallback")
    lib = load_library()
    dev = torch.cuda.current_device() if device is None else int(device)
    h = _handles.get(dev)
    if h is not None:
        return h
    with _lib_lock:
        h = _handles.get(dev)
        if h is not None:
            return h
        out = c_void_p()
        st = lib.si_create(dev, ctypes.byref(out))
        if st != SI_OK:
            _raise(st, "si_create")
        h = out.value
        st = lib.si_set_allocator(h, ctypes.cast(_ALLOC_CB, c_void_p),
                                  ctypes.cast(_FREE_CB, c_void_p), c_void_p(dev))
        if st != SI_OK:
            _raise(st, "si_set_allocator")
        _handles[dev] = h
    return h


def call(name: str, *args) -> None:
    lib = load_library()
    st = getattr(lib, name)(*args)
    if st != SI_OK:
        _raise(st, name)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr(device: torch.device | None = None) -> int:
    """The current CUDA stream of ``device`` (default: the current device) as a
    raw pointer; the raw accessor avoids building a Stream object per call."""
    if _raw_stream is not None:
        idx = device.index if isinstance(device, torch.device) else device
        return _raw_stream(torch.cuda.current_device() if idx is None else int(idx))
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def event_ptr(ev, recorded: bool = False) -> int | None:
    """The ``cudaEvent_t`` of a ``torch.cuda.Event`` for the C ABI (None -> NULL).

    torch creates the underlying CUDA event lazily, at its first ``record``:
    a fresh ``Event()`` has ``cuda_event == 0``, and passing that would make
    the library skip the record and every later ``wait_event`` a no-op.  An
    event the LIBRARY is to record (``recorded=False``) is therefore recorded
    once here on the current stream to create it (the library's record
    replaces that one); an event the CALLER recorded (``recorded=True``, the
    inputs-ready events) must exist already."""
    if ev is None:
        return None
    if not ev.cuda_event:
        if recorded:
            raise ValueError("an input-ready event must be recorded before the call")
        ev.record(torch.cuda.current_stream())
    return ev.cuda_event


def i32_array(values) -> ctypes.Array:
    return (c_int32 * max(len(values), 1))(*values)


def i64_array(values) -> ctypes.Array:
    return (c_int64 * max(len(values), 1))(*values)


def f64_array(values) -> ctypes.Array:
    return (c_double * max(len(values), 1))(*values)


def counter_buf() -> ctypes.Array:
    return (c_int64 * 2)(0, 0)
