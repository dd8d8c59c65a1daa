"""Rasterisation group / L2-policy sweep of the CTA-pair INT8 kernel
(si_ozaki_tune) on 16 residue planes of 16384 x 16384 (one emulated n=16384
product's tensor-core work): burst (best of 3) and sustained (~3 s, power cap)
TOPS per setting, nvidia-smi clocks during the sustained loop.

    python tools/ozaki_tune.py                 # timing sweep -> gpurun_out/ozaki_tune.json
    python tools/ozaki_tune.py --once G A B    # one launch per setting (for ncu DRAM bytes)
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import _lib  # noqa: E402
from int8_yardstick import Clocks, timed  # noqa: E402

SETTINGS = [(16, 0, 0), (8, 0, 0), (4, 0, 0), (32, 0, 0), (16, 1, 2), (8, 1, 2), (4, 1, 2),
            (8, 1, 0), (8, 0, 2)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--once", nargs=3, type=int, default=None)
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--planes", type=int, default=16)
    ap.add_argument("--kernel", default="pair")
    ap.add_argument("--stages", type=int, default=0, help="pair kernel ring depth (3..6)")
    ap.add_argument("--groups", type=str, default=None,
                    help="comma-separated rasterisation groups to sweep (no L2 hints)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    n, planes = args.n, args.planes
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randint(-128, 128, (planes, n, n), dtype=torch.int8, device="cuda", generator=g)
    b = torch.randint(-128, 128, (planes, n, n), dtype=torch.int8, device="cuda", generator=g)
    P.set_ozaki_kernel(args.kernel)
    if args.stages:
        _lib.call("si_ozaki_tune_stages", args.stages)
    ops = 2.0 * n ** 3 * planes
    settings_once = SETTINGS
    if args.groups:
        settings_once = [(int(g), 0, 0) for g in args.groups.split(",")]
    if args.once:
        for s in (settings_once if args.once[0] == 0 else [tuple(args.once)]):
            _lib.call("si_ozaki_tune", *s)
            P.i8_gemm_mod(a, b)
            torch.cuda.synchronize()
        return
    res = {}
    settings = settings_once
    for i, s in enumerate(settings):
        _lib.call("si_ozaki_tune", *s)
        fn = lambda: P.i8_gemm_mod(a, b)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        burst = min(timed(fn, 1) for _ in range(3))
        reps = max(3, int(3000 / burst))
        clk = Clocks()
        sus = timed(fn, reps)
        c = clk.stop()
        res[f"{i}:{s}"] = {"burst_tops": ops / burst / 1e9, "sustained_tops": ops / sus / 1e9,
                       "burst_ms": burst, "sustained_ms": sus, "clocks": c}
        print(s, json.dumps(res[f"{i}:{s}"]), flush=True)
    json.dump(res, open(f"gpurun_out/ozaki_tune_{args.kernel}.json",
                        "w"), indent=1)


if __name__ == "__main__":
    main()
