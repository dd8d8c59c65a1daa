// FP64 peak microbenchmark: DMMA (mma.sync f64 shapes) and DFMA, registers only.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__device__ __forceinline__ void mma_f64(double* c, const double* a, const double* b);

// m8n8k4: a 1, b 1, c 2
template <> __device__ __forceinline__ void mma_f64<0>(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
}
// m16n8k4: a 2, b 1, c 4
template <> __device__ __forceinline__ void mma_f64<1>(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
// m16n8k8: a 4, b 2, c 4
template <> __device__ __forceinline__ void mma_f64<2>(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
// m16n8k16: a 8, b 4, c 4
template <> __device__ __forceinline__ void mma_f64<3>(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
constexpr int kFmas[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};

template <int SHAPE, int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a[8], b[4], c[NACC][4];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = seed * (threadIdx.x - i);
  for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) mma_f64<SHAPE>(c[j], a, b);
  }
  double s = 0;
  for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double acc[NACC];
  double x = seed * threadIdx.x, y = seed + threadIdx.x;
  for (int j = 0; j < NACC; ++j) acc[j] = j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) acc[j] = fma(acc[j], x, y);
  }
  double s = 0;
  for (int j = 0; j < NACC; ++j) s += acc[j];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <typename K>
float time_kernel(K kern, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters, 1e-3);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) kern<<<blocks, threads>>>(out, iters, 1e-3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 3;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 20);
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int blocks = sms * bps, threads = 32 * wpb;
      float ms;
      ms = time_kernel(dmma_loop<0, 8>, blocks, threads, iters, out);
      printf("dmma m8n8k4   warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", wpb, bps, 2.0 * kFmas[0] * 8 * (double)iters * blocks * wpb / (ms * 1e-3) / 1e12);
      ms = time_kernel(dmma_loop<1, 8>, blocks, threads, iters, out);
      printf("dmma m16n8k4  warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", wpb, bps, 2.0 * kFmas[1] * 8 * (double)iters * blocks * wpb / (ms * 1e-3) / 1e12);
      ms = time_kernel(dmma_loop<2, 8>, blocks, threads, iters / 2, out);
      printf("dmma m16n8k8  warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", wpb, bps, 2.0 * kFmas[2] * 8 * (double)(iters / 2) * blocks * wpb / (ms * 1e-3) / 1e12);
      ms = time_kernel(dmma_loop<3, 8>, blocks, threads, iters / 4, out);
      printf("dmma m16n8k16 warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", wpb, bps, 2.0 * kFmas[3] * 8 * (double)(iters / 4) * blocks * wpb / (ms * 1e-3) / 1e12);
      ms = time_kernel(dfma_loop<16>, blocks, threads, iters, out);
      printf("dfma          warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", wpb, bps, 2.0 * 16 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12);
    }
  }
  // sustained: long DMMA run (~4 s)
  {
    int blocks = sms * 2, threads = 256;
    float ms = time_kernel(dmma_loop<0, 8>, blocks, threads, iters * 40, out);
    printf("dmma m8n8k4 sustained (%.0f ms/launch): %.2f TFLOP/s\n", ms, 2.0 * kFmas[0] * 8 * (double)iters * 40 * blocks * 8 / (ms * 1e-3) / 1e12);
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
