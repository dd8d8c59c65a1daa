"""Bitwise A/B of two library builds on emulated products (SI_LIB_PATH selects
the build): writes the products' bytes for a fixed seed so two runs can be
compared (sha256 of each product's bytes).  python tools/crt_ab.py <out.txt>"""
import hashlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_11480_b200 as P  # noqa: E402

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(7)
outs = []
P.set_gemm_backend("ozaki", 16, 128)
for (m, k, n) in ((2048, 2048, 2048), (1500, 3000, 1700), (4096, 1024, 4096)):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(k, n, dtype=torch.float64, device="cuda", generator=g)
    a[3] *= 1e-200
    b[:, 5] *= 1e200
    c = P.mat_mul(a, b, P.MulCounter()).cpu().numpy()
    outs.append(hashlib.sha256(c.tobytes()).hexdigest())
open(sys.argv[1], "w").write("\n".join(outs) + "\n")
