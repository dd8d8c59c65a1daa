"""Achieved bandwidth of the HBM-bound kernels of the path (lincomb, GEMV, the
splitting, the Frobenius reduction) and the n x n x 64 product, at n=16384,
through the C ABI, timed with CUDA events (best of 5 after warm-up).
Writes one JSON object to stdout."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_11480_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists(
    "MEASURED_PEAKS.json") else 7700.0
h, s = _lib.handle(), _lib.stream_ptr()
torch.manual_seed(0)
x = [torch.randn(n, n, dtype=torch.float64, device="cuda") for _ in range(3)]
d = torch.empty(n, n, dtype=torch.float64, device="cuda")
v = torch.randn(n, 1, dtype=torch.float64, device="cuda")
w = torch.empty(n, 1, dtype=torch.float64, device="cuda")
r64 = torch.randn(n, 64, dtype=torch.float64, device="cuda")
o64 = torch.empty(n, 64, dtype=torch.float64, device="cuda")
p2 = torch.empty_like(d)
out = ctypes.c_double()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


res = {"n": n, "hbm_peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)"}
ptrs = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in x])
coef = _lib.f64_array([1.0, -0.5, 0.25])
ld = _lib.i64_array([n, n, n])
sec = timed(lambda: _lib.call("si_lincomb", h, n, n, 1.0, 3, coef, ptrs, ld, d.data_ptr(), n, s))
res["lincomb_3_terms"] = {"bytes": 4 * n * n * 8, "s": sec, "gbs": 4 * n * n * 8 / sec / 1e9}
sec = timed(lambda: _lib.call("si_gemm", h, n, 1, n, 1.0, x[0].data_ptr(), n, v.data_ptr(), 1, 0.0,
                              None, 1, 0.0, w.data_ptr(), 1, 1, None, s))
res["gemv_r1"] = {"bytes": n * n * 8 + 2 * n * 8, "s": sec, "gbs": (n * n * 8) / sec / 1e9}
sec = timed(lambda: _lib.call("si_gemm", h, n, 64, n, 1.0, x[0].data_ptr(), n, r64.data_ptr(), 64,
                              0.0, None, 64, 0.0, o64.data_ptr(), 64, 1, None, s))
res["gemm_n_n_64"] = {"flop": 2 * n * n * 64, "bytes": n * n * 8, "s": sec,
                      "tflops": 2 * n * n * 64 / sec / 1e12, "gbs": n * n * 8 / sec / 1e9}
sec = timed(lambda: _lib.call("si_split_scalar", h, n, x[0].data_ptr(), 3.0, d.data_ptr(),
                              p2.data_ptr(), s))
res["split_scalar"] = {"bytes": 3 * n * n * 8, "s": sec, "gbs": 3 * n * n * 8 / sec / 1e9}
sec = timed(lambda: _lib.call("si_fro_norm", h, n, n, x[0].data_ptr(), n, ctypes.byref(out), s))
res["fro_norm"] = {"bytes": n * n * 8, "s": sec, "gbs": n * n * 8 / sec / 1e9,
                   "note": "includes the host read-back of the scalar"}
for k, val in res.items():
    if isinstance(val, dict) and "gbs" in val:
        val["frac_of_hbm_peak"] = val["gbs"] / peak
print(json.dumps(res, indent=1))
