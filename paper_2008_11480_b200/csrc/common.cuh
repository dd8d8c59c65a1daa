// Shared definitions for the seriesinv B200 kernels and runtime.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

namespace si {

// A dense row-major FP64 matrix view on the device.
struct Mat {
  double* p = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
  __host__ __device__ bool empty() const { return p == nullptr; }
};

// Epilogue of every GEMM: D = alpha * (A @ B) + beta * C + diag * I.
// alpha/beta are +-1 on every reference DAG, so the fused epilogue rounds
// exactly like numpy's "product temporary, then add" (matrix_core.py:101-106
// followed by the element-wise op at the call site).
struct Epilogue {
  double alpha = 1.0;
  double beta = 0.0;
  double diag = 0.0;
  int64_t doff = 0;  // diag*I sits at (i, i + doff): row blocks of a sharded matrix
  const double* c = nullptr;
  int64_t ldc = 0;
  // optional: per-CTA-warp partial sums of squares of the stored values (the
  // fused ||D||_F^2 of newton_schulz.py:328-331); the kernel writes exactly
  // the slots its *_sq_slots() function counts
  double* sq = nullptr;
};

// Panel gate of a product whose right operand B is being gathered row panel
// by row panel (sharded path): rows [bounds[p], bounds[p+1]) of
// B may be read once ready[p] has reached `epoch` (wrap-safe compare).  The
// flags are written by stream memory operations behind the copy of each panel.
constexpr int kMaxPanels = 16;
struct PanelWait {
  const unsigned* ready = nullptr;
  unsigned epoch = 0;
  int npanels = 0;
  int bounds[kMaxPanels + 1] = {};
};

void set_error(const std::string& msg);
const char* get_error();

// Kernel launchers (stream-ordered, no host sync).
cudaError_t launch_gemm_tma(const Mat& A, const Mat& B, Mat& D, const Epilogue& e, cudaStream_t s,
                            const PanelWait* pw = nullptr, const PanelWait* pwa = nullptr);
cudaError_t launch_gemm_generic(const Mat& A, const Mat& B, Mat& D, const Epilogue& e, cudaStream_t s);
cudaError_t launch_gemv(const Mat& A, const Mat& X, Mat& D, const Epilogue& e, cudaStream_t s);
bool tma_eligible(const Mat& A, const Mat& B, const Mat& D, const Epilogue& e);
int64_t gemm_tma_sq_slots(int64_t M, int64_t N);

// D = cdiag * I + sum_i coef[i] * X[i], accumulated in argument order with one
// rounding per term (series_toolkit.py:375-378, numpy temporaries).
constexpr int kMaxLinTerms = 6;
cudaError_t launch_lincomb(Mat& D, double cdiag, int64_t doff, int nterms, const double* coef, const Mat* X,
                           cudaStream_t s);
// D = scale * I  (scale=0 -> zeros)
cudaError_t launch_fill_identity(Mat& D, double scale, cudaStream_t s);
// D = X (strided copy)
cudaError_t launch_copy(Mat& D, const Mat& X, cudaStream_t s);
// D = I - X / alpha (splitting.py:138-140 residual), P = I / alpha
cudaError_t launch_scalar_split(Mat& P, Mat& B, const Mat& A, double alpha, cudaStream_t s);
// D = I - diag(A)^-1 A, P = diag(1/diag(A)) (splitting.py:113-114)
cudaError_t launch_diag_split(Mat& P, Mat& B, const Mat& A, cudaStream_t s);
// Deterministic reductions into a device scalar.
cudaError_t launch_sumsq(const Mat& X, double* out_dev, double* work, cudaStream_t s);
cudaError_t launch_inf_norm(const Mat& X, double* out_dev, double* work, cudaStream_t s);
size_t reduce_work_elems(const Mat& X);
// per-block partial sums of squares only (sumsq_partials() of them, fixed order)
cudaError_t launch_sumsq_partials(const Mat& X, double* part, cudaStream_t s);
int sumsq_partials();
// *out = (accumulate ? *out : 0) + fixed-order sum of part[0..n) (fused-norm slots)
cudaError_t launch_sum_slots(const double* part, int64_t n, double* out, bool accumulate,
                             cudaStream_t s);
// Stream memory operations (driver entry points; executed by the stream's
// front end, no SM involved): *addr = value after prior work, and wait until
// (int32)(*addr - value) >= 0.  Either address may be a peer (IPC) mapping.
cudaError_t stream_write_u32(unsigned* addr, unsigned value, cudaStream_t s);
cudaError_t stream_wait_u32(const unsigned* addr, unsigned value, cudaStream_t s);
// Register-only DMMA throughput of the current device (synchronous).
cudaError_t dmma_peak_tflops(int iters, double* tflops);
// (X + X^T) / 2 into D (splitting.py:73)
cudaError_t launch_symmetrize(Mat& D, const Mat& X, cudaStream_t s);

}  // namespace si
