"""Time the FP64 GEMM's epilogue variants through si_gemm (CUDA events):
plain D = A B, residual D = I - A B, accumulate D = A B + C (C distinct and
C == D in place).  Prints TFLOP/s and a bit-level checksum of each output so
two builds / SI_GEMM_EPI settings can be compared for identical results."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11480_b200 import _lib  # noqa: E402

sizes = [int(x) for x in sys.argv[1:]] or [4096, 16384]
h, s = _lib.handle(), _lib.stream_ptr()
out = {}
for n in sizes:
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    c = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    d = torch.empty_like(a)
    reps = max(3, int(4e13 / (2 * n**3)))

    def run(alpha, beta, cp, diag, dp):
        _lib.call("si_gemm", h, n, n, n, alpha, a.data_ptr(), n, b.data_ptr(), n, beta, cp, n,
                  diag, dp, n, 0, None, s)

    variants = {
        "plain": lambda: run(1.0, 0.0, None, 0.0, d.data_ptr()),
        "residual": lambda: run(-1.0, 0.0, None, 1.0, d.data_ptr()),
        "accumulate": lambda: run(1.0, 1.0, c.data_ptr(), 0.0, d.data_ptr()),
    }
    for name, fn in variants.items():
        fn()
        torch.cuda.synchronize()
        chk = int(d.view(torch.int64).sum().item())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[f"{n}/{name}"] = {"tflops": round(2 * n**3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12, 3),
                              "checksum": chk}
    # in place: D = A B + D, restarted from the same D each rep
    d0 = c.clone()
    d.copy_(d0)
    run(1.0, 1.0, d.data_ptr(), 0.0, d.data_ptr())
    torch.cuda.synchronize()
    out[f"{n}/inplace"] = {"checksum": int(d.view(torch.int64).sum().item())}
print(json.dumps(out))
