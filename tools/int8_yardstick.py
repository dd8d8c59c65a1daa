"""INT8 tensor-core yardstick on this pool's B200s: cuBLASLt int8 GEMM
(torch._int_mm, int8 x int8 -> int32) next to the library's tcgen05 kind::i8
kernel (si_i8_gemm_mod: 16 residue planes, mod m_l epilogue) at the shapes of
the Ozaki-II products -- the measured denominator of the INT8 roofline, the
way MEASURED_PEAKS.json measures bf16 with cuBLAS.

Burst = best of 10 launches; sustained = back to back for ~4 s (power cap).
nvidia-smi clocks sampled during the sustained loops.

Usage: python tools/int8_yardstick.py [--out gpurun_out/int8_yardstick.json]
"""
import argparse
import json
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402


class Clocks:
    def __init__(self):
        self.lines = []
        self.p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,"
                                   "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits",
                                   "-lms", "200"], stdout=subprocess.PIPE, text=True)
        self.t = threading.Thread(target=lambda: [self.lines.append(l) for l in self.p.stdout],
                                  daemon=True)
        self.t.start()

    def stop(self):
        self.p.terminate()
        self.t.join(timeout=2)
        sm = sorted(float(l.split(",")[0]) for l in self.lines if l.count(",") == 2)
        pw = sorted(float(l.split(",")[1]) for l in self.lines if l.count(",") == 2)
        cap = sum("Active" in l for l in self.lines)
        return {"sm_mhz_median": sm[len(sm) // 2] if sm else None,
                "power_w_median": pw[len(pw) // 2] if pw else None,
                "power_cap_samples": cap, "samples": len(sm)}


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def measure(fn, ops):
    fn()
    torch.cuda.synchronize()
    burst = min(timed(fn, 1) for _ in range(10))
    reps = max(3, int(4000 / burst))
    clk = Clocks()
    sus = timed(fn, reps)
    c = clk.stop()
    return {"burst_ms": burst, "burst_tops": ops / burst / 1e9, "sustained_ms": sus,
            "sustained_tops": ops / sus / 1e9, "reps": reps, "clocks": c}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/int8_yardstick.json")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    res = {"gpu": torch.cuda.get_device_name(0)}
    for n in (8192, 16384):
        a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda", generator=g)
        b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda", generator=g)
        bt = b.t()  # column-major B for cuBLASLt (TN)
        r = measure(lambda: torch._int_mm(a, bt), 2.0 * n ** 3)
        res[f"cublaslt_int_mm_{n}"] = r
        print(n, "cublasLt", json.dumps(r), flush=True)
        del b, bt
        planes = 16 if n == 8192 else 4
        a3 = torch.randint(-128, 128, (planes, n, n), dtype=torch.int8, device="cuda", generator=g)
        b3 = torch.randint(-128, 128, (planes, n, n), dtype=torch.int8, device="cuda", generator=g)
        for kernel in ("pair", "single", "multicast"):
            P.set_ozaki_kernel(kernel)
            r = measure(lambda: P.i8_gemm_mod(a3, b3), 2.0 * n ** 3 * planes)
            res[f"si_i8_gemm_mod_{kernel}_{planes}x{n}"] = r
            print(n, "si_i8", kernel, json.dumps(r), flush=True)
        P.set_ozaki_kernel("auto")
        del a3, b3, a
        torch.cuda.empty_cache()
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
