"""Wave-lockstep A/B of the DMMA GEMM (gemm_tma.cu): times n x n x n products
with CUDA events and prints a bitwise checksum of D, so runs with
SI_GEMM_LOCKSTEP=0 / 1 (separate processes: the switch is read once) can be
compared for speed and identical output.

    python tools/gemm_lockstep_probe.py 4096 16384 32768
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11480_b200 import _lib  # noqa: E402

h, s = _lib.handle(), _lib.stream_ptr()
for n in [int(x) for x in sys.argv[1:]] or [16384]:
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    d = torch.empty_like(a)
    reps = max(2, min(10, int(2e14 / (2 * n**3))))

    def run():
        # the residual form of the hot path: D = I - A B (alpha=-1, diag=1)
        _lib.call("si_gemm", h, n, n, n, -1.0, a.data_ptr(), n, b.data_ptr(), n, 0.0, None, n,
                  1.0, d.data_ptr(), n, 0, None, s)

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    chk = int(d.view(torch.int64).sum().item()) & ((1 << 64) - 1)
    print(f"n={n} reps={reps} ms={ms:.3f} tflops={2 * n**3 / ms / 1e9:.3f} checksum={chk:016x}",
          flush=True)
    del a, b, d
    torch.cuda.empty_cache()
