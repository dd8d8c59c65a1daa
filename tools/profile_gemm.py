"""Small driver for ncu: a few FP64 GEMMs (TMA/DMMA kernel) at n x n x n, plus one
fused-epilogue residual GEMM, through the C ABI."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11480_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.manual_seed(0)
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
d = torch.empty_like(a)
h, s = _lib.handle(), _lib.stream_ptr()
for i in range(reps):
    _lib.call("si_gemm", h, n, n, n, -1.0, a.data_ptr(), n, b.data_ptr(), n, 1.0, a.data_ptr(), n,
              1.0 if i % 2 else 0.0, d.data_ptr(), n, 0, None, s)
torch.cuda.synchronize()
print("ok", float(d[0, 0]))
