// Setup-path kernels: fused symmetry check + symmetrize,
// blocked Cholesky positive-definiteness check, device power iteration.
#pragma once
#include "engine.hpp"

namespace si {

// (X + X^T) / 2 into D (D may equal X) in one pass over tile pairs, and
// out3 = {||X - X^T||_F, ||X||_F, #non-finite entries} (device scalars;
// fixed-order reductions).  `work` holds symcheck_work_elems() doubles.
cudaError_t launch_symcheck(Mat& D, const Mat& X, double* work, double* out3, cudaStream_t s);
size_t symcheck_work_elems();

// splitting.py:76-98: true iff the Cholesky of (a + a^T)/2 finds every pivot
// > tol, tol = 1e-12 ||a||_inf when default_tol (else pivot_tol).  Blocked
// right-looking (128-wide panels): diagonal block in shared memory, panel by
// forward substitution, trailing update on the DMMA GEMM.  Synchronises the
// stream (every 16 panels, to stop early on a failed pivot).
bool cholesky_pd(Ctx& c, const MV& a, double pivot_tol, bool default_tol, int64_t* fail_index,
                 double* fail_pivot);

// matrix_core.py:183-239 state, device-resident between iterations.
enum : int { kPowerRunning = 0, kPowerConverged = 1, kPowerNullSpace = 2, kPowerMaxIter = 3 };
struct PowerState {
  double est, prev, best;
  int64_t iters;
  int streak, has_prev, status, pad;
};
// `iters` iterations of { y = A x; est = ||y||; the reference's stop rules;
// x = y / est } queued without any host synchronisation; iterations after a
// stop (status != running) do nothing but the product.
cudaError_t launch_power_iters(const Mat& A, double* x, double* y, double* part, PowerState* st,
                               double tol, int64_t max_iter, int iters, cudaStream_t s);

}  // namespace si
