// Small / irregular FP64 GEMM (DMMA), skinny GEMV, and the O(n^2) element-wise
// and reduction kernels of the seriesinv hot path.
//
//  * gemm_generic: any shape, stride and alignment (reference tests use n=2..8;
//    config 1 uses n=64).  64x64 CTA tile, 4 warps of 32x32, DMMA m8n8k4.
//  * gemv: n x r products with r <= 4 (mat_vec, matrix_core.py:109-114) --
//    HBM-bound, one warp per row, fixed-order shuffle reduction.
//  * lincomb: the Lin instruction of a lowered plan (series_toolkit.py:375-378)
//    and the free sums of the step bodies; one rounding per term, in order.
//  * split kernels: splitting.py:113-114 and :138-140 evaluated on device.
//  * sumsq / inf_norm: deterministic two-level reductions (matrix_core.py:154-172).
#include "common.cuh"

namespace si {
namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double apply_epi(double acc, double alpha, double beta, double cval) {
  double v = (alpha == 1.0) ? acc : (alpha == -1.0 ? -acc : __dmul_rn(alpha, acc));
  if (beta != 0.0) v = __dadd_rn(v, beta == 1.0 ? cval : __dmul_rn(beta, cval));
  return v;
}

constexpr int GB = 64;   // CTA tile (square)
constexpr int GK = 16;   // k slab
constexpr int GPAD = 4;  // row padding (doubles)

__global__ void __launch_bounds__(128) gemm_generic_kernel(
    const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
    double* __restrict__ D, int64_t ldd, const double* __restrict__ C, int64_t ldc, int64_t M,
    int64_t N, int64_t K, double alpha, double beta, double diag, int64_t doff) {
  __shared__ double As[GB][GK + GPAD];
  __shared__ double Bs[GK][GB + GPAD];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 1, wn = warp & 1;
  const int g = lane >> 2, t = lane & 3;
  const int64_t m0 = (int64_t)blockIdx.y * GB, n0 = (int64_t)blockIdx.x * GB;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int64_t k0 = 0; k0 < K; k0 += GK) {
    // 64x16 A slab and 16x64 B slab, 8 elements of each per thread.
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = tid + i * 128;
      const int ar = idx / GK, ac = idx % GK;
      const int64_t gr = m0 + ar, gc = k0 + ac;
      As[ar][ac] = (gr < M && gc < K) ? A[gr * lda + gc] : 0.0;
      const int br = idx / GB, bc = idx % GB;
      const int64_t hr = k0 + br, hc = n0 + bc;
      Bs[br][bc] = (hr < K && hc < N) ? B[hr * ldb + hc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = As[wm * 32 + mi * 8 + g][kk + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = Bs[kk + t][wn * 32 + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int64_t row = m0 + wm * 32 + mi * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = n0 + wn * 32 + ni * 8 + 2 * t + h;
        if (col >= N) continue;
        double cv = (beta != 0.0) ? C[row * ldc + col] : 0.0;
        double v = apply_epi(acc[mi][ni][h], alpha, beta, cv);
        if (diag != 0.0 && row + doff == col) v = __dadd_rn(v, diag);
        D[row * ldd + col] = v;
      }
    }
  }
}

// 16-byte read-only load that does not allocate in L1 (the matrix row is
// streamed once; X stays cached)
__device__ __forceinline__ double2 ldg_stream2(const double2* p) {
  double2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

// D[i, j] = alpha * sum_k A[i,k] X[k,j] + beta*C[i,j] + diag*[i==j], j < NR <= 4.
// One warp per row.  VEC: the row is read as 16-byte pairs, eight per lane in
// flight (A 16-byte aligned, lda and K even) -- the row stream is the whole
// cost, so memory-level parallelism is what sets the bandwidth.
template <int NR, bool VEC>
__global__ void __launch_bounds__(256) gemv_kernel(const double* __restrict__ A, int64_t lda,
                                                   const double* __restrict__ X, int64_t ldx,
                                                   double* __restrict__ D, int64_t ldd,
                                                   const double* __restrict__ C, int64_t ldc,
                                                   int64_t M, int64_t K, double alpha,
                                                   double beta, double diag, int64_t doff) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= M) return;
  double s[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) s[j] = 0.0;
  const double* a = A + row * lda;
  if (VEC) {
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const int64_t K2 = K >> 1;
    auto step = [&](double2 av, int64_t k2) {
      const int64_t k = 2 * k2;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        s[j] = fma(av.x, __ldg(X + k * ldx + j), s[j]);
        s[j] = fma(av.y, __ldg(X + (k + 1) * ldx + j), s[j]);
      }
    };
    int64_t k2 = lane;
    for (; k2 + 32 * 7 < K2; k2 += 256) {
      double2 av[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) av[u] = ldg_stream2(a2 + k2 + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; ++u) step(av[u], k2 + 32 * u);
    }
    for (; k2 < K2; k2 += 32) step(ldg_stream2(a2 + k2), k2);
  } else {
    for (int64_t k = lane; k < K; k += 32) {
      const double av = __ldg(a + k);
#pragma unroll
      for (int j = 0; j < NR; ++j) s[j] = fma(av, __ldg(X + k * ldx + j), s[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < NR; ++j) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], off);
  }
  if (lane < NR) {
    double v = s[0];
#pragma unroll
    for (int j = 1; j < NR; ++j)
      if (lane == j) v = s[j];
    const double cv = (beta != 0.0) ? C[row * ldc + lane] : 0.0;
    v = apply_epi(v, alpha, beta, cv);
    if (diag != 0.0 && row + doff == lane) v = __dadd_rn(v, diag);
    D[row * ldd + lane] = v;
  }
}

struct LinArgs {
  const double* x[kMaxLinTerms];
  int64_t ldx[kMaxLinTerms];
  double coef[kMaxLinTerms];
};

__global__ void lincomb_kernel(double* __restrict__ D, int64_t ldd, int64_t M, int64_t N,
                               double cdiag, int64_t doff, int nterms, LinArgs args) {
  const int64_t total = M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i % N;
    double acc = (r + doff == c) ? cdiag : 0.0;
    for (int j = 0; j < nterms; ++j) {
      const double xv = args.x[j][r * args.ldx[j] + c];
      const double term = (args.coef[j] == 1.0) ? xv : __dmul_rn(args.coef[j], xv);
      acc = __dadd_rn(acc, term);
    }
    D[r * ldd + c] = acc;
  }
}

__global__ void fill_identity_kernel(double* __restrict__ D, int64_t ldd, int64_t M, int64_t N,
                                     double scale) {
  const int64_t total = M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i % N;
    D[r * ldd + c] = (r == c) ? scale : 0.0;
  }
}

__global__ void copy_kernel(double* __restrict__ D, int64_t ldd, const double* __restrict__ X,
                            int64_t ldx, int64_t M, int64_t N) {
  const int64_t total = M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i % N;
    D[r * ldd + c] = X[r * ldx + c];
  }
}

// P = I/alpha, B = I - A/alpha: numpy rounds identity(n)/alpha and a/alpha,
// then the subtraction (splitting.py:138-140).
__global__ void scalar_split_kernel(double* __restrict__ P, int64_t ldp, double* __restrict__ Bm,
                                    int64_t ldb, const double* __restrict__ A, int64_t lda,
                                    int64_t n, double alpha) {
  const int64_t total = n * n;
  const double pinv = __ddiv_rn(1.0, alpha);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i % n;
    const double q = __ddiv_rn(A[r * lda + c], alpha);
    Bm[r * ldb + c] = __dsub_rn(r == c ? 1.0 : 0.0, q);
    if (P) P[r * ldp + c] = (r == c) ? pinv : 0.0;
  }
}

// P = diag(1/d), B = I - A / d[:, None] (splitting.py:113-114)
__global__ void diag_split_kernel(double* __restrict__ P, int64_t ldp, double* __restrict__ Bm,
                                  int64_t ldb, const double* __restrict__ A, int64_t lda,
                                  int64_t n) {
  const int64_t total = n * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i % n;
    const double d = A[r * lda + r];
    const double q = __ddiv_rn(A[r * lda + c], d);
    Bm[r * ldb + c] = __dsub_rn(r == c ? 1.0 : 0.0, q);
    if (P) P[r * ldp + c] = (r == c) ? __ddiv_rn(1.0, d) : 0.0;
  }
}

__global__ void symmetrize_kernel(double* __restrict__ D, int64_t ldd, const double* __restrict__ X,
                                  int64_t ldx, int64_t n) {
  const int64_t total = n * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i % n;
    D[r * ldd + c] = __dmul_rn(__dadd_rn(X[r * ldx + c], X[c * ldx + r]), 0.5);
  }
}

constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 1184;  // 8 x 148 SMs

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[RED_THREADS / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (threadIdx.x < RED_THREADS / 32) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
  }
  return r;
}

__global__ void __launch_bounds__(RED_THREADS) sumsq_partial(const double* __restrict__ X,
                                                            int64_t ldx, int64_t M, int64_t N,
                                                            double* __restrict__ part) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ldx == N && !(reinterpret_cast<uintptr_t>(X) & 15u)) {
    // contiguous: 16-byte streaming loads, four per thread in flight
    const double2* x2 = reinterpret_cast<const double2*>(X);
    const int64_t n2 = (M * N) >> 1;
    int64_t i = tid;
    for (; i + 3 * stride < n2; i += 4 * stride) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ldg_stream2(x2 + i + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s = fma(v[u].x, v[u].x, s);
        s = fma(v[u].y, v[u].y, s);
      }
    }
    for (; i < n2; i += stride) {
      const double2 v = ldg_stream2(x2 + i);
      s = fma(v.x, v.x, s);
      s = fma(v.y, v.y, s);
    }
    if (tid == 0 && ((M * N) & 1)) s = fma(X[M * N - 1], X[M * N - 1], s);
  } else {
    // strided rows: one block per row at a time
    for (int64_t r = blockIdx.x; r < M; r += gridDim.x)
      for (int64_t c = threadIdx.x; c < N; c += blockDim.x) {
        const double v = X[r * ldx + c];
        s = fma(v, v, s);
      }
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS) sum_final(const double* __restrict__ part, int n,
                                                        double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
}

// Row sums of |X| (one warp per row), then a fixed-order max.
__global__ void __launch_bounds__(RED_THREADS) rowabs_kernel(const double* __restrict__ X,
                                                            int64_t ldx, int64_t M, int64_t N,
                                                            double* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (RED_THREADS / 32) + (threadIdx.x >> 5);
  if (r >= M) return;
  double s = 0.0;
  for (int64_t c = lane; c < N; c += 32) s += fabs(X[r * ldx + c]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) rows[r] = s;
}

__global__ void __launch_bounds__(RED_THREADS) max_final(const double* __restrict__ v, int64_t n,
                                                        double* __restrict__ out) {
  __shared__ double sh[RED_THREADS];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, v[i]);
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int w = RED_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// Register-only DMMA throughput probe (roofline denominator).
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters, double seed) {
  const int lane = threadIdx.x & 31;
  double a = seed * (lane + 1), b = seed * (lane + 2);
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int ew_grid(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

cudaError_t launch_gemm_generic(const Mat& A, const Mat& B, Mat& D, const Epilogue& e,
                                cudaStream_t s) {
  dim3 grid((unsigned)((D.cols + GB - 1) / GB), (unsigned)((D.rows + GB - 1) / GB));
  gemm_generic_kernel<<<grid, 128, 0, s>>>(A.p, A.ld, B.p, B.ld, D.p, D.ld, e.c, e.ldc, D.rows,
                                           D.cols, A.cols, e.alpha, e.beta, e.diag, e.doff);
  return cudaGetLastError();
}

cudaError_t launch_gemv(const Mat& A, const Mat& X, Mat& D, const Epilogue& e, cudaStream_t s) {
  const unsigned grid = (unsigned)((D.rows + 7) / 8);
  // pairs only pay for long rows; short rows keep the one-element-per-lane order
  const bool vec = A.cols >= 256 && ((reinterpret_cast<uintptr_t>(A.p) & 15u) == 0) &&
                   !(A.ld & 1) && !(A.cols & 1);
  auto go = [&](auto kern) {
    kern<<<grid, 256, 0, s>>>(A.p, A.ld, X.p, X.ld, D.p, D.ld, e.c, e.ldc, D.rows, A.cols, e.alpha,
                              e.beta, e.diag, e.doff);
  };
  switch (D.cols) {
    case 1: vec ? go(gemv_kernel<1, true>) : go(gemv_kernel<1, false>); break;
    case 2: vec ? go(gemv_kernel<2, true>) : go(gemv_kernel<2, false>); break;
    case 3: vec ? go(gemv_kernel<3, true>) : go(gemv_kernel<3, false>); break;
    default: vec ? go(gemv_kernel<4, true>) : go(gemv_kernel<4, false>); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_lincomb(Mat& D, double cdiag, int64_t doff, int nterms, const double* coef, const Mat* X,
                           cudaStream_t s) {
  if (nterms > kMaxLinTerms) return cudaErrorInvalidValue;
  LinArgs args{};
  for (int i = 0; i < nterms; ++i) {
    args.x[i] = X[i].p;
    args.ldx[i] = X[i].ld;
    args.coef[i] = coef[i];
  }
  lincomb_kernel<<<ew_grid(D.rows * D.cols), 256, 0, s>>>(D.p, D.ld, D.rows, D.cols, cdiag, doff, nterms,
                                                          args);
  return cudaGetLastError();
}

cudaError_t launch_fill_identity(Mat& D, double scale, cudaStream_t s) {
  fill_identity_kernel<<<ew_grid(D.rows * D.cols), 256, 0, s>>>(D.p, D.ld, D.rows, D.cols, scale);
  return cudaGetLastError();
}

cudaError_t launch_copy(Mat& D, const Mat& X, cudaStream_t s) {
  if (D.ld == D.cols && X.ld == X.cols)
    return cudaMemcpyAsync(D.p, X.p, sizeof(double) * D.rows * D.cols, cudaMemcpyDeviceToDevice, s);
  copy_kernel<<<ew_grid(D.rows * D.cols), 256, 0, s>>>(D.p, D.ld, X.p, X.ld, D.rows, D.cols);
  return cudaGetLastError();
}

cudaError_t launch_scalar_split(Mat& P, Mat& B, const Mat& A, double alpha, cudaStream_t s) {
  scalar_split_kernel<<<ew_grid(A.rows * A.rows), 256, 0, s>>>(P.p, P.ld, B.p, B.ld, A.p, A.ld,
                                                               A.rows, alpha);
  return cudaGetLastError();
}

cudaError_t launch_diag_split(Mat& P, Mat& B, const Mat& A, cudaStream_t s) {
  diag_split_kernel<<<ew_grid(A.rows * A.rows), 256, 0, s>>>(P.p, P.ld, B.p, B.ld, A.p, A.ld,
                                                             A.rows);
  return cudaGetLastError();
}

cudaError_t launch_symmetrize(Mat& D, const Mat& X, cudaStream_t s) {
  symmetrize_kernel<<<ew_grid(X.rows * X.rows), 256, 0, s>>>(D.p, D.ld, X.p, X.ld, X.rows);
  return cudaGetLastError();
}

cudaError_t dmma_peak_tflops(int iters, double* tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  cudaError_t err = cudaMalloc(&out, 256 * sizeof(double));
  if (err != cudaSuccess) return err;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 2 * sms;
  dmma_peak_kernel<<<blocks, 256>>>(out, iters / 10 + 1, 1e-3);  // warm-up
  cudaEventRecord(e0);
  dmma_peak_kernel<<<blocks, 256>>>(out, iters, 1e-3);
  cudaEventRecord(e1);
  err = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err == cudaSuccess) err = cudaGetLastError();
  // 8 DMMA.8x8x4 (256 FMA) per iteration per warp, 8 warps per block
  *tflops = 2.0 * 256.0 * 8.0 * (double)iters * blocks * 8.0 / (ms * 1e-3) / 1e12;
  return err;
}

size_t reduce_work_elems(const Mat& X) {
  return (size_t)(X.rows > RED_BLOCKS ? X.rows : RED_BLOCKS);
}

cudaError_t launch_sumsq(const Mat& X, double* out_dev, double* work, cudaStream_t s) {
  sumsq_partial<<<RED_BLOCKS, RED_THREADS, 0, s>>>(X.p, X.ld, X.rows, X.cols, work);
  sum_final<<<1, RED_THREADS, 0, s>>>(work, RED_BLOCKS, out_dev);
  return cudaGetLastError();
}

int sumsq_partials() { return RED_BLOCKS; }

// *out = (accumulate ? *out : 0) + sum of part[0..n) in a fixed order
__global__ void __launch_bounds__(RED_THREADS) sum_slots_kernel(const double* __restrict__ part,
                                                               int64_t n, double* __restrict__ out,
                                                               int accumulate) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = accumulate ? *out + s : s;
}

cudaError_t launch_sum_slots(const double* part, int64_t n, double* out, bool accumulate,
                             cudaStream_t s) {
  sum_slots_kernel<<<1, RED_THREADS, 0, s>>>(part, n, out, accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_sumsq_partials(const Mat& X, double* part, cudaStream_t s) {
  sumsq_partial<<<RED_BLOCKS, RED_THREADS, 0, s>>>(X.p, X.ld, X.rows, X.cols, part);
  return cudaGetLastError();
}

cudaError_t launch_inf_norm(const Mat& X, double* out_dev, double* work, cudaStream_t s) {
  const unsigned grid = (unsigned)((X.rows + RED_THREADS / 32 - 1) / (RED_THREADS / 32));
  rowabs_kernel<<<grid, RED_THREADS, 0, s>>>(X.p, X.ld, X.rows, X.cols, work);
  max_final<<<1, RED_THREADS, 0, s>>>(work, X.rows, out_dev);
  return cudaGetLastError();
}

}  // namespace si
