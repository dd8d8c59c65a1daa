"""One emulated FP64 product (and one DMMA product) at size n -- for ncu launch lists."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
mod = int(sys.argv[2]) if len(sys.argv) > 2 else 16
torch.manual_seed(0)
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
with P.gemm_backend("ozaki", moduli=mod, min_dim=1024):
    for _ in range(2):
        c = P.mat_mul(a, b, P.MulCounter())
with P.gemm_backend("dmma"):
    d = P.mat_mul(a, b, P.MulCounter())
torch.cuda.synchronize()
print("rel diff", ((c - d).norm() / d.norm()).item())
