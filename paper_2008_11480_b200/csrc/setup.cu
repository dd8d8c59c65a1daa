// Setup-path kernels: the fused symmetry check +
// symmetrize pass of splitting.py:67-73, the positive-definiteness check of
// splitting.py:76-98 as a blocked right-looking Cholesky whose trailing
// updates run on the DMMA GEMM, and the norm-ratio power iteration of
// matrix_core.py:183-239 with device-side convergence tests.
#include "setup.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>

namespace si {
namespace {

// ---------------------------------------------------------------------------
// symmetry check + symmetrize: one pass over tile pairs (i, j) / (j, i)
// ---------------------------------------------------------------------------

constexpr int ST = 32;            // tile edge
constexpr int SYM_THREADS = 256;  // 32 x 8
constexpr int SYM_BLOCKS = 1184;  // 8 x 148 SMs

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Each block owns tile pairs p = blockIdx.x, blockIdx.x + gridDim.x, ... (i <= j)
// and writes its partial sums of ||X - X^T||_F^2, ||X||_F^2 and the count of
// non-finite entries to part[3 b .. 3 b + 2] (fixed assignment: deterministic).
// D may equal X: a pair's two tiles are read into shared memory before either
// is written, and no other block touches them.
__global__ void __launch_bounds__(SYM_THREADS) symcheck_kernel(double* D, int64_t ldd,
                                                               const double* X, int64_t ldx,
                                                               int64_t n, double* part) {
  __shared__ double t0[ST][ST + 1], t1[ST][ST + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t T = (n + ST - 1) / ST;
  double asym = 0.0, fro = 0.0, bad = 0.0;
  for (int64_t p = blockIdx.x; p < T * T; p += gridDim.x) {
    const int64_t i = p / T, j = p % T;
    if (i > j) continue;
    for (int r = ty; r < ST; r += 8) {
      const int64_t gr = i * ST + r, gc = j * ST + tx;
      t0[r][tx] = (gr < n && gc < n) ? X[gr * ldx + gc] : 0.0;
      const int64_t hr = j * ST + r, hc = i * ST + tx;
      t1[r][tx] = (hr < n && hc < n) ? X[hr * ldx + hc] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < ST; r += 8) {
      const int64_t gr = i * ST + r, gc = j * ST + tx;
      if (gr < n && gc < n) {
        const double v = t0[r][tx], w = t1[tx][r];  // X[gr][gc], X[gc][gr]
        const double d = __dsub_rn(v, w);
        if (i == j) {
          asym = fma(d, d, asym);  // both (r, c) and (c, r) lie in this tile
          fro = fma(v, v, fro);
          bad += isfinite(v) ? 0.0 : 1.0;
        } else {
          asym = fma(2.0 * d, d, asym);  // the pair's mirror element has the same |d|
          fro = fma(v, v, fma(w, w, fro));
          bad += (isfinite(v) ? 0.0 : 1.0) + (isfinite(w) ? 0.0 : 1.0);
        }
        // (a + a.T) / 2.0 with numpy's rounding (splitting.py:73)
        t0[r][tx] = __dmul_rn(__dadd_rn(v, w), 0.5);  // only this thread reads t0[r][tx]
      }
    }
    __syncthreads();
    for (int r = ty; r < ST; r += 8) {
      const int64_t gr = i * ST + r, gc = j * ST + tx;
      if (gr < n && gc < n) D[gr * ldd + gc] = t0[r][tx];
      const int64_t hr = j * ST + r, hc = i * ST + tx;
      if (i != j && hr < n && hc < n) D[hr * ldd + hc] = t0[tx][r];
    }
    __syncthreads();
  }
  __shared__ double red[3][SYM_THREADS / 32];
  asym = warp_sum(asym);
  fro = warp_sum(fro);
  bad = warp_sum(bad);
  if (tx == 0) {
    red[0][ty] = asym;
    red[1][ty] = fro;
    red[2][ty] = bad;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int w = 0; w < SYM_THREADS / 32; ++w) s += red[threadIdx.x][w];
    part[3 * blockIdx.x + threadIdx.x] = s;
  }
}

// fixed-order sums of the per-block partials: out[0] = ||X - X^T||_F,
// out[1] = ||X||_F, out[2] = non-finite count
__global__ void __launch_bounds__(SYM_THREADS) symcheck_final(const double* part, int nb,
                                                              double* out) {
  __shared__ double red[3][SYM_THREADS / 32];
  double s[3] = {0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    for (int k = 0; k < 3; ++k) s[k] += part[3 * b + k];
  for (int k = 0; k < 3; ++k) {
    const double v = warp_sum(s[k]);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int w = 0; w < SYM_THREADS / 32; ++w) v += red[threadIdx.x][w];
    out[threadIdx.x] = threadIdx.x < 2 ? sqrt(v) : v;
  }
}

// ---------------------------------------------------------------------------
// blocked Cholesky (positive-definiteness check)
// ---------------------------------------------------------------------------

constexpr int CH_THREADS = 512;

// Unblocked Cholesky of the nb x nb diagonal block at (k0, k0) in shared
// memory, with the reference's pivot test d <= tol -> not PD
// (splitting.py:88-90); L (lower, zeros above) goes to Lkk.  status[0] = 1 and
// status[1] = global pivot index on failure; later steps then return at once.
__global__ void __launch_bounds__(CH_THREADS) chol_diag_kernel(const double* A, int64_t lda,
                                                               int64_t k0, int nb,
                                                               const double* norm_dev,
                                                               double tol_factor, double tol_abs,
                                                               double* Lkk, int* status,
                                                               double* fail_pivot) {
  extern __shared__ double L[];  // nb x (nb + 1)
  if (*(volatile int*)status) return;
  const int ld = nb + 1;
  const double tol = norm_dev ? tol_factor * *norm_dev : tol_abs;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int r = e / nb, c = e % nb;
    L[r * ld + c] = A[(k0 + r) * lda + k0 + c];
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double d = L[j * ld + j];
    if (!(d > tol)) {  // d <= tol, or NaN
      if (threadIdx.x == 0) {
        status[0] = 1;
        status[1] = (int)(k0 + j);
        *fail_pivot = d;
      }
      return;  // every thread read the same d: uniform exit
    }
    const double ljj = sqrt(d);
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) L[i * ld + j] = __ddiv_rn(L[i * ld + j], ljj);
    if (threadIdx.x == 0) L[j * ld + j] = ljj;
    __syncthreads();
    // trailing lower triangle: L[i][c] -= L[i][j] L[c][j], j < c <= i
    const int m = nb - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int ii = e / m, cc = e % m;
      if (cc > ii) continue;
      const int i = j + 1 + ii, c = j + 1 + cc;
      L[i * ld + c] = fma(-L[i * ld + j], L[c * ld + j], L[i * ld + c]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int r = e / nb, c = e % nb;
    Lkk[e] = c <= r ? L[r * ld + c] : 0.0;
  }
}

// W = A[k0+nb:, k0:k0+nb] L^-T by forward substitution, one warp per row
// (nb = 128: four columns per lane; the solved x_j is broadcast by shuffle).
template <int NB>
__global__ void __launch_bounds__(256) chol_trsm_kernel(const double* A, int64_t lda, int64_t k0,
                                                        int64_t m, const double* Lkk, double* W,
                                                        const int* status) {
  extern __shared__ double Ls[];  // L^T: Ls[j NB + c] = L[c][j] (lanes read consecutive c)
  if (*(volatile const int*)status) return;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Ls[(e % NB) * NB + e / NB] = Lkk[e];
  __syncthreads();
  constexpr int Q = NB / 32;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int64_t row = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); row < m;
       row += (int64_t)gridDim.x * warps) {
    const double* a = A + (k0 + NB + row) * lda + k0;
    double x[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) x[q] = a[q * 32 + lane];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
#pragma unroll 4
      for (int jj = 0; jj < 32; ++jj) {
        const int j = q * 32 + jj;
        if (lane == jj) x[q] = __ddiv_rn(x[q], Ls[j * NB + j]);
        const double xj = __shfl_sync(0xffffffffu, x[q], jj);
#pragma unroll
        for (int qq = q; qq < Q; ++qq) {
          const int c = qq * 32 + lane;
          if (c > j) x[qq] = fma(-xj, Ls[j * NB + c], x[qq]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) W[row * NB + q * 32 + lane] = x[q];
  }
}

// WT (cols x rows, ld ldt) = W^T (W: rows x cols, ld cols)
__global__ void transpose_kernel(const double* W, int64_t rows, int64_t cols, double* WT,
                                 int64_t ldt, const int* status) {
  __shared__ double t[ST][ST + 1];
  if (status && *(volatile const int*)status) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.y * ST, c0 = (int64_t)blockIdx.x * ST;
  for (int r = ty; r < ST; r += 8)
    if (r0 + r < rows && c0 + tx < cols) t[r][tx] = W[(r0 + r) * cols + c0 + tx];
  __syncthreads();
  for (int c = ty; c < ST; c += 8)
    if (c0 + c < cols && r0 + tx < rows) WT[(c0 + c) * ldt + r0 + tx] = t[tx][c];
}

// ---------------------------------------------------------------------------
// power iteration (matrix_core.py:183-239)
// ---------------------------------------------------------------------------

// One iteration's scalar logic after y = A x and the partial sums of y^2: the
// reference's est / streak / restart / max_iter rules, then x = y / est.
__global__ void __launch_bounds__(1024) power_update_kernel(const double* part, int nparts,
                                                            const double* y, double* x, int64_t n,
                                                            PowerState* st, double tol,
                                                            int64_t max_iter) {
  __shared__ double red[32];
  __shared__ int go;
  if (threadIdx.x == 0) go = st->status == kPowerRunning;
  __syncthreads();
  if (!go) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  __shared__ double est_sh;
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w];
    const double est = sqrt(v);
    st->iters += 1;
    est_sh = est;
    if (est == 0.0) {
      st->status = kPowerNullSpace;  // the host restarts with a fresh vector
    } else {
      st->best = est;
      if (st->has_prev && fabs(est - st->prev) <= tol * est) {
        st->streak += 1;
        if (st->streak >= 3) st->status = kPowerConverged;
      } else {
        st->streak = 0;
      }
      st->prev = est;
      st->has_prev = 1;
      if (st->status == kPowerRunning && st->iters >= max_iter) st->status = kPowerMaxIter;
    }
    st->est = est;
  }
  __syncthreads();
  if (st->status != kPowerRunning) return;
  const double est = est_sh;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = __ddiv_rn(y[i], est);
}

}  // namespace

cudaError_t launch_symcheck(Mat& D, const Mat& X, double* work, double* out3, cudaStream_t s) {
  symcheck_kernel<<<SYM_BLOCKS, SYM_THREADS, 0, s>>>(D.p, D.ld, X.p, X.ld, X.rows, work);
  symcheck_final<<<1, SYM_THREADS, 0, s>>>(work, SYM_BLOCKS, out3);
  return cudaGetLastError();
}

size_t symcheck_work_elems() { return 3 * (size_t)SYM_BLOCKS; }

bool cholesky_pd(Ctx& c, const MV& a, double pivot_tol, bool default_tol, int64_t* fail_index,
                 double* fail_pivot) {
  Handle* h = c.h;
  const int64_t n = a.v.rows;
  if (n == 0) return true;
  const int64_t ld = n + (n & 1);  // even: every panel offset stays 16-byte aligned for TMA
  MV w = alloc(c, n, ld);
  w.v.cols = n;
  // (a + a.T) / 2 into the workspace (splitting.py:84), and ||a||_inf for the
  // default pivot floor 1e-12 ||a||_inf (splitting.py:86-87)
  MV sc = alloc(c, 1, (int64_t)symcheck_work_elems() + 8);
  check(launch_symcheck(w.v, a.v, sc.v.p, sc.v.p + symcheck_work_elems(), c.s), "symmetrize");
  double* norm_dev = nullptr;
  MV red;  // kept alive to the end: the diagonal kernels read the norm
  if (default_tol) {
    red = alloc(c, 1, (int64_t)reduce_work_elems(w.v) + 1);
    norm_dev = red.v.p + reduce_work_elems(w.v);
    check(launch_inf_norm(w.v, norm_dev, red.v.p, c.s), "inf norm");
  }
  constexpr int NB = 128;
  MV lkk = alloc(c, NB, NB);
  MV stat = alloc(c, 1, 2);  // int status[2] + fail pivot (as doubles)
  int* status = reinterpret_cast<int*>(stat.v.p);
  double* piv = stat.v.p + 1;
  check(cudaMemsetAsync(stat.v.p, 0, 2 * sizeof(double), c.s), "memset");
  MV wpanel = alloc(c, n, NB);
  MV wt = alloc(c, NB, ld);
  {  // opt-in shared memory of the two kernels, once per device
    static std::atomic<uint64_t> attr_set{0};
    const int dev = c.h->device;
    if (dev >= 64 || !(attr_set.load() & (1ull << dev))) {
      check(cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 NB * (NB + 1) * 8),
            "cudaFuncSetAttribute");
      check(cudaFuncSetAttribute(chol_trsm_kernel<NB>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, NB * NB * 8),
            "cudaFuncSetAttribute");
      if (dev < 64) attr_set.fetch_or(1ull << dev);
    }
  }
  int hstat[4] = {0, 0, 0, 0};
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int nb = (int)std::min<int64_t>(NB, n - k0);
    chol_diag_kernel<<<1, CH_THREADS, nb * (nb + 1) * 8, c.s>>>(
        w.v.p, ld, k0, nb, norm_dev, 1e-12, pivot_tol, lkk.v.p, status, piv);
    h->launches += 1;
    const int64_t m = n - k0 - nb;
    if (m > 0) {
      // nb == NB here (only the last block can be short)
      chol_trsm_kernel<NB><<<148 * 4, 256, NB * NB * 8, c.s>>>(w.v.p, ld, k0, m, lkk.v.p,
                                                               wpanel.v.p, status);
      const int64_t ldt = m + (m & 1);
      dim3 tg((unsigned)((NB + ST - 1) / ST), (unsigned)((m + ST - 1) / ST));
      transpose_kernel<<<tg, 256, 0, c.s>>>(wpanel.v.p, m, NB, wt.v.p, ldt, status);
      h->launches += 2;
      check(cudaGetLastError(), "cholesky panel");
      // trailing update A22 -= W W^T on the DMMA GEMM (in place: D == C).  Only
      // the lower triangle is ever read again (the diagonal blocks and the
      // panels below them), so large trailing matrices are updated in row
      // strips, each up to its own last column: ~(1 + 1/strips)/2 of the
      // product (the k order per entry is unchanged: same pivots, bitwise).
      double* a22p = w.v.p + (k0 + NB) * ld + k0 + NB;
      const int64_t strips = m >= 4096 ? std::min<int64_t>(8, m / 2048) : 1;
      const int64_t sr = ((m + strips - 1) / strips + NB - 1) / NB * NB;
      for (int64_t i0 = 0; i0 < m; i0 += sr) {
        const int64_t i1 = std::min(m, i0 + sr);
        MV a22 = view(a22p + i0 * ld, i1 - i0, i1, ld);
        MV wl = view(wpanel.v.p + i0 * NB, i1 - i0, NB, NB);
        MV wr = view(wt.v.p, NB, i1, ldt);
        gemm(c, a22, wl, wr, -1.0, &a22, 1.0, 0.0, false);
      }
    }
    check(cudaGetLastError(), "cholesky diag");
    // early exit: look at the status every 16 panels
    if (((k0 / NB) & 15) == 15 || k0 + NB >= n) {
      check(cudaMemcpyAsync(hstat, stat.v.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.s),
            "memcpy");
      check(cudaStreamSynchronize(c.s), "sync");
      if (hstat[0]) break;
    }
  }
  if (hstat[0]) {
    double pv;
    std::memcpy(&pv, &hstat[2], sizeof(double));
    if (fail_index) *fail_index = hstat[1];
    if (fail_pivot) *fail_pivot = pv;
    return false;
  }
  if (fail_index) *fail_index = -1;
  return true;
}

cudaError_t launch_power_iters(const Mat& A, double* x, double* y, double* part, PowerState* st,
                               double tol, int64_t max_iter, int iters, cudaStream_t s) {
  Mat X{x, A.cols, 1, 1};
  Mat Y{y, A.rows, 1, 1};
  Epilogue e;
  for (int k = 0; k < iters; ++k) {
    cudaError_t err = launch_gemv(A, X, Y, e, s);
    if (err != cudaSuccess) return err;
    err = launch_sumsq_partials(Y, part, s);
    if (err != cudaSuccess) return err;
    power_update_kernel<<<1, 1024, 0, s>>>(part, sumsq_partials(), y, x, A.rows, st, tol,
                                           max_iter);
  }
  return cudaGetLastError();
}

}  // namespace si
