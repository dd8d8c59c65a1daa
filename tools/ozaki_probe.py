"""GPU probe of the Ozaki-II INT8 tensor-core path (csrc/ozaki.cu).

1. the INT8 tcgen05 kernel alone vs exact integer products (cuBLAS FP64 of
   small integers is exact),
2. emulated FP64 products vs an extended-precision reference (numpy
   longdouble) next to the DMMA product's error,
3. timing at n = 4096 / 16384: emulated product, its INT8 kernel (TOPS), DMMA.

Usage: python tools/ozaki_probe.py [--big] [--moduli 16]
"""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402
from paper_2008_11480_b200 import _lib  # noqa: E402


def gemm(a, b, backend, moduli=16):
    with P.gemm_backend(backend, moduli=moduli, min_dim=128):
        c = P.mat_mul(a, b, P.MulCounter())
    return c


def check_i8():
    out = []
    mods = P.ozaki_moduli(16)
    g = torch.Generator(device="cuda").manual_seed(1)
    for (planes, m, n, kp) in [(1, 128, 256, 128), (3, 300, 520, 256), (2, 1000, 777, 1024),
                               (16, 512, 512, 4096)]:
        a = torch.randint(-128, 128, (planes, m, kp), dtype=torch.int8, device="cuda", generator=g)
        bt = torch.randint(-128, 128, (planes, n, kp), dtype=torch.int8, device="cuda", generator=g)
        r = P.i8_gemm_mod(a, bt)
        torch.cuda.synchronize()
        ok = True
        for l in range(planes):
            ref = torch.remainder(a[l].double() @ bt[l].double().T, mods[l]).to(torch.uint8)
            bad = (ref != r[l]).sum().item()
            ok &= bad == 0
            if bad:
                idx = (ref != r[l]).nonzero()[:4].tolist()
                out.append(dict(case=(planes, m, n, kp), plane=l, bad=bad, first=idx))
        out.append(dict(case=(planes, m, n, kp), exact=ok))
    return out


def ext_ref(a, b):
    return (a.cpu().numpy().astype(np.longdouble) @ b.cpu().numpy().astype(np.longdouble))


def check_accuracy(moduli):
    rows = []
    rng = np.random.default_rng(0)
    cases = {
        "gauss": lambda n: (rng.standard_normal((n, n)), rng.standard_normal((n, n))),
        "wide_rows": lambda n: (rng.standard_normal((n, n)) * np.exp2(rng.integers(-30, 30, (n, 1))),
                                rng.standard_normal((n, n))),
        "wide_entries": lambda n: (rng.standard_normal((n, n)) * np.exp2(rng.integers(-20, 20, (n, n))),
                                   rng.standard_normal((n, n)) * np.exp2(rng.integers(-20, 20, (n, n)))),
        "spd_residual": lambda n: _residual_pair(rng, n),
    }
    for name, mk in cases.items():
        for n in (384, 768):
            a_np, b_np = mk(n)
            a = torch.from_numpy(a_np).cuda()
            b = torch.from_numpy(b_np).cuda()
            ref = ext_ref(a, b)
            absab = (np.abs(a_np) @ np.abs(b_np))
            res = {}
            for be, mo in [("dmma", 16), ("ozaki", moduli), ("ozaki", 14), ("ozaki", 12)]:
                c = gemm(a, b, be, mo).cpu().numpy().astype(np.longdouble)
                err = np.abs(c - ref)
                key = be if be == "dmma" else f"ozaki{mo}"
                res[key] = dict(
                    rel_fro=float(np.linalg.norm((c - ref).astype(np.float64)) /
                                  np.linalg.norm(ref.astype(np.float64))),
                    max_comp=float(np.max(err / np.maximum(absab, 1e-300))),
                )
            rows.append(dict(case=name, n=n, **res))
    return rows


def _residual_pair(rng, n):
    g = rng.standard_normal((2 * n, n))
    a = g.T @ g / (2 * n) + 1e-3 * np.eye(n)
    p = np.eye(n) / np.abs(a).sum(1).max()
    f = np.eye(n) - p @ a
    return f, f


def timing(n, moduli, reps=3):
    torch.manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    h = _lib.handle()
    lib = _lib.load_library()
    out = {}
    for be in ("ozaki", "dmma"):
        with P.gemm_backend(be, moduli=moduli, min_dim=1024):
            P.mat_mul(a, b, P.MulCounter())
            torch.cuda.synchronize()
            lib.si_profile_begin(h)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                P.mat_mul(a, b, P.MulCounter())
            e1.record()
            torch.cuda.synchronize()
            import ctypes
            ms, fl, ng, nl = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
            lib.si_profile_end(h, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(ng), ctypes.byref(nl))
            ims, iops, il = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
            lib.si_profile_i8(h, ctypes.byref(ims), ctypes.byref(iops), ctypes.byref(il))
            t = e0.elapsed_time(e1) / reps
            out[be] = dict(ms_per_product=t, fp64_tflops=2 * n ** 3 / t / 1e9,
                           i8_ms=ims.value / max(il.value, 1),
                           i8_tops=(iops.value / (ims.value * 1e-3) / 1e12) if il.value else None)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--moduli", type=int, default=16)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    res = {"i8": check_i8()}
    print(json.dumps(res["i8"]), flush=True)
    res["accuracy"] = check_accuracy(args.moduli)
    for r in res["accuracy"]:
        print(json.dumps(r), flush=True)
    res["timing"] = {}
    for n in ((4096, 16384) if args.big else (4096,)):
        res["timing"][n] = timing(n, args.moduli)
        print(n, json.dumps(res["timing"][n]), flush=True)
    json.dump(res, open("gpurun_out/ozaki_probe.json", "w"), indent=1)
