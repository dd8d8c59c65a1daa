// DMMA m8n8k4 throughput when the fragments come from shared memory (as in the
// resident kernels), by warp tile and warps per SM sub-partition.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_lds dmma_lds.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// each warp: `iters` products of a 32-deep K over an (8 MT) x (8 NT) tile,
// fragments loaded one k-step ahead from a 32 x 32 shared tile (no swizzle:
// A rows g, cols t; B rows t, cols g -- 2-way conflicts at most)
template <int MT, int NT>
__global__ void lds_dmma(double* out, int iters) {
  __shared__ double tileA[64 * 36], tileB[64 * 36];
  for (int i = threadIdx.x; i < 64 * 36; i += blockDim.x) {
    tileA[i] = 1e-3 * (i % 7);
    tileB[i] = 1e-3 * (i % 5);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[MT][NT][2] = {};
  for (int it = 0; it < iters; ++it) {
    double af[2][MT], bf[2][NT];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) af[0][mi] = tileA[(mi * 8 + g) * 36 + t];
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) bf[0][ni] = tileB[t * 36 + ni * 8 + g];
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      const int cur = (kk >> 2) & 1, nxt = cur ^ 1;
      if (kk + 4 < 32) {
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) af[nxt][mi] = tileA[(mi * 8 + g) * 36 + kk + 4 + t];
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) bf[nxt][ni] = tileB[(kk + 4 + t) * 36 + ni * 8 + g];
      }
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[cur][mi], bf[cur][ni]);
    }
  }
  double s = 0;
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) s += acc[mi][ni][0] + acc[mi][ni][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int MT, int NT>
void run(int warps_per_block, int blocks_per_sm, int sms, double* out) {
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = blocks_per_sm * sms;
  lds_dmma<MT, NT><<<blocks, 32 * warps_per_block>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  lds_dmma<MT, NT><<<blocks, 32 * warps_per_block>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * blocks * warps_per_block * (double)iters * MT * NT * 8 * 8 * 32;
  printf("tile %2dx%-2d warps/SM %2d (%d x %d blocks): %6.2f TFLOP/s\n", 8 * MT, 8 * NT,
         warps_per_block * blocks_per_sm, warps_per_block, blocks_per_sm, flops / ms / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  for (int bps : {2, 4, 5}) run<4, 2>(2, bps, sms, out);   // C2 warp tile (32 x 16)
  for (int bps : {2, 4, 5}) run<2, 4>(2, bps, sms, out);   // 16 x 32
  for (int bps : {2, 4, 5}) run<1, 4>(4, bps, sms, out);   // 8 x 32
  for (int bps : {2, 4, 5}) run<4, 1>(4, bps, sms, out);   // 32 x 8
  for (int bps : {2, 4}) run<2, 2>(4, bps, sms, out);      // 16 x 16
  for (int bps : {2, 4}) run<4, 4>(1, bps * 2, sms, out);  // 32 x 32
  for (int bps : {2, 4}) run<2, 8>(1, bps * 2, sms, out);  // 16 x 64
  cudaFree(out);
  return 0;
}
