"""Feasibility probe: does CRT / residue work on a second stream overlap an
INT8 GEMM at the power cap?  Stream g runs the INT8 kernel on 16 residue planes
of 16384^2 (~46 ms); stream x runs emulated products 16384 x 512 by 512 x 16384
(their time is scaling + residues + the full-size CRT; their INT8 GEMMs are
small).  Times g alone, x alone and both together (CUDA events, after warm-up).

    python tools/overlap_probe.py
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(0)
    a3 = torch.randint(-128, 128, (16, n, n), dtype=torch.int8, device="cuda", generator=g)
    b3 = torch.randint(-128, 128, (16, n, n), dtype=torch.int8, device="cuda", generator=g)
    k = 512
    xa = torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g)
    xb = torch.randn(k, n, dtype=torch.float64, device="cuda", generator=g)
    P.set_gemm_backend("ozaki", 16, 128)
    sg, sx = torch.cuda.Stream(), torch.cuda.Stream()
    reps_x = 8

    def run_g():
        with torch.cuda.stream(sg):
            P.i8_gemm_mod(a3, b3)

    def run_x():
        with torch.cuda.stream(sx):
            for _ in range(reps_x):
                P.mat_mul(xa, xb, P.MulCounter())

    def timed(fns):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in (sg, sx):
            s.wait_event(e0)
        for f in fns:
            f()
        for s in (sg, sx):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for f in (run_g, run_x):
        f()
    torch.cuda.synchronize()
    res = {}
    for rep in range(3):
        res.setdefault("g_alone_ms", []).append(timed([run_g]))
        res.setdefault("x_alone_ms", []).append(timed([run_x]))
        res.setdefault("both_ms", []).append(timed([run_g, run_x]))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
