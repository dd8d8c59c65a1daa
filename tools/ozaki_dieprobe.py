"""Probe: the single-CTA INT8 kernel with its 16 planes split between the two
dies by %smid (si_ozaki_tune group 2^21 | 16) vs the default raster --
equality of the result bytes, sustained TOPS at the power cap (alternating).

    python tools/ozaki_dieprobe.py [--once]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import _lib  # noqa: E402
from int8_yardstick import Clocks, timed  # noqa: E402

DEFAULT, SPLIT = (16, 0, 0), ((1 << 21) | 16, 0, 0)

torch.cuda.set_device(0)
n, planes = 16384, 16
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randint(-128, 128, (planes, n, n), dtype=torch.int8, device="cuda", generator=g)
b = torch.randint(-128, 128, (planes, n, n), dtype=torch.int8, device="cuda", generator=g)
P.set_ozaki_kernel("single")
if "--once" in sys.argv:
    for s in (DEFAULT, SPLIT):
        _lib.call("si_ozaki_tune", *s)
        P.i8_gemm_mod(a, b)
    torch.cuda.synchronize()
    sys.exit(0)
_lib.call("si_ozaki_tune", *DEFAULT)
ref = P.i8_gemm_mod(a, b)
_lib.call("si_ozaki_tune", *SPLIT)
got = P.i8_gemm_mod(a, b)
print("split result equal:", bool(torch.equal(ref, got)), flush=True)
del ref, got
ops = 2.0 * n ** 3 * planes
res = {}
for i, s in enumerate([DEFAULT, SPLIT, DEFAULT, SPLIT]):
    _lib.call("si_ozaki_tune", *s)
    fn = lambda: P.i8_gemm_mod(a, b)  # noqa: E731
    fn()
    torch.cuda.synchronize()
    reps = 60
    clk = Clocks()
    sus = timed(fn, reps)
    c = clk.stop()
    res[f"{i}:{'split' if s == SPLIT else 'default'}"] = {"sustained_tops": ops / sus / 1e9, "ms": sus, "clocks": c}
    print(i, s, json.dumps(res[f"{i}:{'split' if s == SPLIT else 'default'}"]), flush=True)
_lib.call("si_ozaki_tune", *DEFAULT)
json.dump(res, open("gpurun_out/ozaki_dieprobe.json", "w"), indent=1)
