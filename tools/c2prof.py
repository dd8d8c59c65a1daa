import sys, torch
sys.path.insert(0, ".")
import paper_2008_11480_b200 as P
from paper_2008_11480_b200 import configs
a_np, b_np = configs.c2_batched(batch=2048)
a, b = P.as_device(a_np), P.as_device(b_np)
pre, res = P.batched_scalar_split(a)
for _ in range(2):
    P.batched_composite_richardson(a, b, pre, res, pre, res, torch.zeros_like(b), (2, 3), 2, 10)
torch.cuda.synchronize(); print("ok")
