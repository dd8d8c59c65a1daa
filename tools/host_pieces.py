"""Per-piece host cost of the Python call path (diagnostics)."""
import sys, time, torch, ctypes
sys.path.insert(0, ".")
import paper_2008_11480_b200 as P
from paper_2008_11480_b200 import _lib
x = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
def t(name, fn, n=2000):
    fn(); s = time.perf_counter()
    for _ in range(n): fn()
    print(f"{name:40s} {(time.perf_counter()-s)/n*1e6:6.2f} us")
t("current_stream().cuda_stream", lambda: torch.cuda.current_stream().cuda_stream)
t("_lib.stream_ptr(x.device)", lambda: _lib.stream_ptr(x.device))
t("torch._C._cuda_getCurrentRawStream(0)", lambda: torch._C._cuda_getCurrentRawStream(0))
t("empty_like", lambda: torch.empty_like(x))
t("reshape+contiguous", lambda: x.reshape(1, 64, 64).contiguous())
t("as_device", lambda: P.as_device(x))
t("counter_buf", lambda: _lib.counter_buf())
t("handle", lambda: _lib.handle(0))
t("x.device.index", lambda: x.device.index)
t("data_ptr", lambda: x.data_ptr())
t("current_device", lambda: torch.cuda.current_device())
