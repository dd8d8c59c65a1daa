"""Host cost of one config-1 batched call (diagnostics): the Python wrapper
vs the C-ABI call alone.  python tools/c1host.py"""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2008_11480_b200 as P
from paper_2008_11480_b200 import configs
a_np, b_np = configs.c1_dense_small()
a, b = P.as_device(a_np), P.as_device(b_np)
alpha = float(torch.max(torch.sum(torch.abs(a), dim=1)))
eye = torch.eye(64, dtype=torch.float64, device="cuda")
p0, f0, t0 = eye / alpha, eye - a / alpha, torch.zeros_like(b)
for _ in range(5): P.batched_ns_richardson(a, b, p0, f0, t0, 3, 30)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200): P.batched_ns_richardson(a, b, p0, f0, t0, 3, 1)
h = time.perf_counter() - t
torch.cuda.synchronize(); tt = time.perf_counter() - t
print(f"host per call {h/200*1e6:.1f} us; wall per call (1 iteration) {tt/200*1e6:.1f} us")

# split: the C-ABI call alone vs the Python wrapper around it
from paper_2008_11480_b200 import _lib
p_in, f_in, th_in = p0.reshape(1, 64, 64).contiguous(), f0.reshape(1, 64, 64).contiguous(), t0.reshape(1, 64)
p_io, f_io, th_io = torch.empty_like(p_in), torch.empty_like(f_in), torch.empty_like(th_in)
h = _lib.handle(0)
buf = _lib.counter_buf()
sp = _lib.stream_ptr(a.device)
args = (h, 1, 64, a.data_ptr(), b.data_ptr(), 3, None, 0, None, 0, 1, p_in.data_ptr(), f_in.data_ptr(),
        th_in.data_ptr(), p_io.data_ptr(), f_io.data_ptr(), th_io.data_ptr(), buf, sp)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200): _lib.call("si_batched_ns_richardson_ex", *args)
hc = time.perf_counter() - t
torch.cuda.synchronize()
print(f"C-ABI call alone {hc/200*1e6:.1f} us")
