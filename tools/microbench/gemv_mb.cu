// GEMV (n x n times n x 1, FP64) variants: achieved HBM bandwidth, CUDA events,
// best of 10.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 gemv_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

// V0: one warp per row, one element per lane per iteration
__global__ void __launch_bounds__(256) v0(const double* __restrict__ A, const double* __restrict__ x,
                                          double* __restrict__ y, int n) {
  const int lane = threadIdx.x & 31;
  const long row = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  double s = 0.0;
  const double* a = A + row * n;
  for (long k = lane; k < n; k += 32) s = fma(__ldg(a + k), __ldg(x + k), s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  if (!lane) y[row] = s;
}

// V1: pairs, four per lane in flight
__global__ void __launch_bounds__(256) v1(const double* __restrict__ A, const double* __restrict__ x,
                                          double* __restrict__ y, int n) {
  const int lane = threadIdx.x & 31;
  const long row = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  double s = 0.0;
  const double2* a2 = reinterpret_cast<const double2*>(A + row * n);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const long K2 = n >> 1;
  for (long k2 = lane; k2 < K2; k2 += 128) {
    double2 av[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = k2 + 32 * u < K2;
      av[u] = ok ? __ldg(a2 + k2 + 32 * u) : make_double2(0, 0);
      xv[u] = ok ? __ldg(x2 + k2 + 32 * u) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s = fma(av[u].x, xv[u].x, s);
      s = fma(av[u].y, xv[u].y, s);
    }
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  if (!lane) y[row] = s;
}

// V2: pairs, persistent grid-stride over rows (no tail wave), 4 in flight
__global__ void __launch_bounds__(256) v2(const double* __restrict__ A, const double* __restrict__ x,
                                          double* __restrict__ y, int n) {
  const int lane = threadIdx.x & 31;
  const long K2 = n >> 1;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  for (long row = (long)blockIdx.x * 8 + (threadIdx.x >> 5); row < n; row += (long)gridDim.x * 8) {
    double s = 0.0;
    const double2* a2 = reinterpret_cast<const double2*>(A + row * n);
    for (long k2 = lane; k2 < K2; k2 += 128) {
      double2 av[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = k2 + 32 * u < K2;
        av[u] = ok ? __ldg(a2 + k2 + 32 * u) : make_double2(0, 0);
        xv[u] = ok ? __ldg(x2 + k2 + 32 * u) : make_double2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s = fma(av[u].x, xv[u].x, s);
        s = fma(av[u].y, xv[u].y, s);
      }
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
    if (!lane) y[row] = s;
  }
}

// V3: pairs, unroll 8 (8 x 16 B per lane in flight)
__global__ void __launch_bounds__(256) v3(const double* __restrict__ A, const double* __restrict__ x,
                                          double* __restrict__ y, int n) {
  const int lane = threadIdx.x & 31;
  const long row = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  double s = 0.0;
  const double2* a2 = reinterpret_cast<const double2*>(A + row * n);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const long K2 = n >> 1;
  long k2 = lane;
  for (; k2 + 32 * 7 < K2; k2 += 256) {
    double2 av[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      av[u] = __ldg(a2 + k2 + 32 * u);
      xv[u] = __ldg(x2 + k2 + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = fma(av[u].x, xv[u].x, s);
      s = fma(av[u].y, xv[u].y, s);
    }
  }
  for (; k2 < K2; k2 += 32) {
    const double2 av = __ldg(a2 + k2), xv = __ldg(x2 + k2);
    s = fma(av.x, xv.x, s);
    s = fma(av.y, xv.y, s);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  if (!lane) y[row] = s;
}

// V4: like V3 but A loaded with L1::no_allocate streaming hint (ld.global.nc.L1::no_allocate)
__device__ __forceinline__ double2 ldg_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__global__ void __launch_bounds__(256) v4(const double* __restrict__ A, const double* __restrict__ x,
                                          double* __restrict__ y, int n) {
  const int lane = threadIdx.x & 31;
  const long row = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  double s = 0.0;
  const double2* a2 = reinterpret_cast<const double2*>(A + row * n);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const long K2 = n >> 1;
  long k2 = lane;
  for (; k2 + 32 * 7 < K2; k2 += 256) {
    double2 av[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      av[u] = ldg_stream(a2 + k2 + 32 * u);
      xv[u] = __ldg(x2 + k2 + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = fma(av[u].x, xv[u].x, s);
      s = fma(av[u].y, xv[u].y, s);
    }
  }
  for (; k2 < K2; k2 += 32) {
    const double2 av = ldg_stream(a2 + k2), xv = __ldg(x2 + k2);
    s = fma(av.x, xv.x, s);
    s = fma(av.y, xv.y, s);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  if (!lane) y[row] = s;
}

int main() {
  for (int n : {4096, 16384, 32768}) {
    double *A, *x, *y;
    cudaMalloc(&A, (size_t)n * n * 8);
    cudaMalloc(&x, (size_t)n * 8);
    cudaMalloc(&y, (size_t)n * 8);
    cudaMemset(A, 0, (size_t)n * n * 8);
    cudaMemset(x, 0, (size_t)n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
      launch();
      cudaDeviceSynchronize();
      float best = 1e30f;
      for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("n=%d %s %.1f us %.0f GB/s\n", n, name, best * 1e3, (double)n * n * 8 / (best * 1e-3) / 1e9);
    };
    const unsigned g = (n + 7) / 8;
    timeit("v0 scalar", [&] { v0<<<g, 256>>>(A, x, y, n); });
    timeit("v1 pairs4", [&] { v1<<<g, 256>>>(A, x, y, n); });
    timeit("v2 persistent", [&] { v2<<<148 * 8, 256>>>(A, x, y, n); });
    timeit("v3 pairs8", [&] { v3<<<g, 256>>>(A, x, y, n); });
    timeit("v4 pairs8 stream", [&] { v4<<<g, 256>>>(A, x, y, n); });
    cudaFree(A);
    cudaFree(x);
    cudaFree(y);
  }
  return 0;
}
