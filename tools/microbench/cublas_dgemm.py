"""cuBLAS DGEMM yardstick (torch.matmul fp64) at the BASELINE sizes; CUDA-event timed."""
import torch, time, json
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (1024, 2048, 4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    reps = max(1, int(2e13 / (2 * n**3)))
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[n] = 2 * n**3 / (ms * 1e-3) / 1e12
    print(f"cublas dgemm n={n}: {ms:.3f} ms  {res[n]:.2f} TFLOP/s", flush=True)
print(json.dumps(res))
