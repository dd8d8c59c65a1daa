// Dependent-chain latency of DMMA.8x8x4 and of LDS.64 on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, int n) {
  double c0 = threadIdx.x * 1e-3, c1 = 0.5, a = 1.0000001, b = 0.9999999;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  __shared__ double sm[64];
  sm[threadIdx.x] = c0;
  __syncwarp();
  int idx = threadIdx.x;
  double s = 0;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(sm + idx)));
    idx = ((int)v & 31) ^ threadIdx.x;  // dependent address
    s += v;
  }
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; }
  out[threadIdx.x] = c0 + c1 + s;
}

int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1024); cudaMallocManaged(&cyc, 16);
  const int n = 4096;
  chain<<<1, 32>>>(out, cyc, n); cudaDeviceSynchronize();
  chain<<<1, 32>>>(out, cyc, n); cudaDeviceSynchronize();
  printf("DMMA dependent-chain latency: %.1f cycles\n", (double)cyc[0] / n);
  printf("LDS.64 dependent-chain latency (incl. int convert): %.1f cycles\n", (double)cyc[1] / n);
  return 0;
}
