"""Time the library's FP64 GEMM (si_gemm, TMA/DMMA kernel) against cuBLAS DGEMM
(torch.matmul) with CUDA events; prints TFLOP/s per size."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11480_b200 import _lib  # noqa: E402

sizes = [int(x) for x in sys.argv[1:]] or [2048, 4096, 8192, 16384]
h, s = _lib.handle(), _lib.stream_ptr()
for n in sizes:
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    d = torch.empty_like(a)
    reps = max(2, int(3e13 / (2 * n**3)))

    def ours():
        _lib.call("si_gemm", h, n, n, n, 1.0, a.data_ptr(), n, b.data_ptr(), n, 0.0, None, n, 0.0,
                  d.data_ptr(), n, 0, None, s)

    def cublas():
        torch.matmul(a, b, out=d)

    res = {}
    for name, fn in (("ours", ours), ("cublas", cublas)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = 2 * n**3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(f"n={n}: ours {res['ours']:.2f} TFLOP/s   cublas {res['cublas']:.2f} TFLOP/s", flush=True)
