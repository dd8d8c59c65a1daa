"""Time the config-2 resident kernel alone for a few batch sizes (diagnostics):
python tools/c2time.py [iters]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import configs  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
for batch in (2048, 4096, 16384):
    a_np, b_np = configs.c2_batched(batch=batch)
    a, b = P.as_device(a_np), P.as_device(b_np)
    pre, res = P.batched_scalar_split(a)
    th = torch.zeros_like(b)
    for _ in range(2):
        P.batched_composite_richardson(a, b, pre, res, pre, res, th, (2, 3), 2, iters)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        P.batched_composite_richardson(a, b, pre, res, pre, res, th, (2, 3), 2, iters)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"batch {batch} iters {iters}: {ms:.3f} ms, {iters / ms * 1e3:.0f} iters/s, "
          f"{batch * iters / ms / 1e3:.0f} system-iters/ms")
