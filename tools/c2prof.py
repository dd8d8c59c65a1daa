"""ncu driver: the config-2 resident kernel at the bench shape (16384 systems
x 50 iterations per launch); launch 2 is the one to capture (-s 1 -c 1)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import configs  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
a_np, b_np = configs.c2_batched(batch=batch)
a, b = P.as_device(a_np), P.as_device(b_np)
pre, res = P.batched_scalar_split(a)
for _ in range(2):
    P.batched_composite_richardson(a, b, pre, res, pre, res, torch.zeros_like(b), (2, 3), 2, iters)
torch.cuda.synchronize()
print("ok")
