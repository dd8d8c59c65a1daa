"""Time of the device PD check (blocked Cholesky, csrc/setup.cu) at size n."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
torch.manual_seed(0)
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n + 1e-3 * torch.eye(n, dtype=torch.float64, device="cuda")
del g
for _ in range(2):
    ok = P.is_positive_definite(a)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    ok = P.is_positive_definite(a)
torch.cuda.synchronize()
print(f"n={n} pd={ok} {1e3 * (time.perf_counter() - t0) / 3:.1f} ms per check")
