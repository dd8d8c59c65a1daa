"""Host<->device copy bandwidth of the e2e path's buffers: pinned H2D, D2H, and
both at once on two streams (10.75 GB in / 4.3 GB out per C4 step)."""
import json
import sys

import torch

torch.cuda.set_device(0)
n = 16384
nbytes = n * n * 8
h_in = [torch.empty(n, n, dtype=torch.float64).pin_memory() for _ in range(2)]
h_out = [torch.empty(n, n, dtype=torch.float64).pin_memory() for _ in range(2)]
d = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(2)]
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    for s in (up, down):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def h2d():
    with torch.cuda.stream(up):
        for i in range(2):
            d[i].copy_(h_in[i], non_blocking=True)


def d2h():
    with torch.cuda.stream(down):
        for i in range(2):
            h_out[i].copy_(d[i], non_blocking=True)


def both():
    h2d()
    d2h()


res = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    fn()
    t = min(timed(fn) for _ in range(3))
    res[name] = {"s": t, "GBps_each_direction": 2 * nbytes / t / 1e9}
print(json.dumps(res))
