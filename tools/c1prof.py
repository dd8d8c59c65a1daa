"""ncu driver: the config-1 resident kernel (n=64, 30 iterations per launch)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import configs  # noqa: E402

a_np, b_np = configs.c1_dense_small()
a, b = P.as_device(a_np), P.as_device(b_np)
alpha = float(torch.max(torch.sum(torch.abs(a), dim=1)))
eye = torch.eye(64, dtype=torch.float64, device="cuda")
for _ in range(3):
    P.batched_ns_richardson(a, b, eye / alpha, eye - a / alpha, torch.zeros_like(b), 3, 30)
torch.cuda.synchronize()
print("ok")
