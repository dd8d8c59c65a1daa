"""FP64 GEMM through si_gemm with padded leading dimensions (A, B, C, D all
stored with ld = n + pad), timed with CUDA events -- for checking whether
power-of-two row strides cost L2 reuse (run under ncu for DRAM bytes)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11480_b200 import _lib  # noqa: E402

n = int(sys.argv[1])
pad = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ld = n + pad
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, ld, dtype=torch.float64, device="cuda", generator=g)
b = torch.randn(n, ld, dtype=torch.float64, device="cuda", generator=g)
d = torch.empty(n, ld, dtype=torch.float64, device="cuda")
h, s = _lib.handle(), _lib.stream_ptr()


def run():
    _lib.call("si_gemm", h, n, n, n, -1.0, a.data_ptr(), ld, b.data_ptr(), ld, 0.0, None, ld, 1.0,
              d.data_ptr(), ld, 0, None, s)


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
print(f"n={n} ld={ld}: {2 * n**3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12:.3f} TFLOP/s")
