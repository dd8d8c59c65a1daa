/* A non-Python host of the C ABI (include/seriesinv_b200.h): what a C / C++ /
 * Go (cgo) / Java (JNI) caller of the drop-in boundary does.  Device memory
 * comes from the CUDA runtime; every computation is a library call.
 *
 *   A (n x n SPD), b  ->  si_split_scalar     (splitting.py:124-146)
 *                     ->  si_initial_series   (newton_schulz.py:127-147)
 *   k = 1..steps      ->  si_plain_richardson (theta - P (A theta - b))
 *                     ->  si_ns_step order 3  (newton_schulz.py:150-174)
 *
 * Checks on the host: the Richardson mismatch ||A theta - b|| contracts, the
 * residual ||F||_F (si_fro_norm) falls as F_k = F_{k-1}^3, F = I - G A holds,
 * the step with the products emulated on the INT8 tensor cores matches FP64 DMMA,
 * the counters tick like MulCounter (3 mmm + 2 mvm per step after the init),
 * and a bad argument returns SI_EINVAL with a message.  Exit status 0 = pass. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "seriesinv_b200.h"

#define CK(x)                                                                   \
  do {                                                                          \
    int st_ = (x);                                                              \
    if (st_ != SI_OK) {                                                         \
      fprintf(stderr, "%s failed (%d): %s\n", #x, st_, si_last_error());       \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

static double lcg(unsigned long long* s) {
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return ((double)(*s >> 11) / 9007199254740992.0) - 0.5;
}

int main(void) {
  const int64_t n = 256;
  const int steps = 6;
  const size_t mat = (size_t)n * n * sizeof(double), vec = (size_t)n * sizeof(double);
  double *hA = malloc(mat), *hM = malloc(mat), *hb = malloc(vec), *hx = malloc(vec);
  double *hG = malloc(mat), *hF = malloc(mat);
  unsigned long long seed = 2008;
  /* A = M^T M / n + I/2 (SPD), b random */
  for (int64_t i = 0; i < n * n; ++i) hM[i] = lcg(&seed);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k) s += hM[k * n + i] * hM[k * n + j];
      hA[i * n + j] = s / (double)n + (i == j ? 0.5 : 0.0);
    }
  for (int64_t i = 0; i < n; ++i) hb[i] = lcg(&seed);
  double alpha = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double r = 0.0;
    for (int64_t j = 0; j < n; ++j) r += fabs(hA[i * n + j]);
    if (r > alpha) alpha = r;
  }
  /* alpha = ||A||_inf >= lambda_max: rho(I - A / alpha) < 1 */

  double *dA, *dP, *dB, *dG, *dF, *dG2, *dF2, *db, *dx, *dx2;
  cudaMalloc((void**)&dA, mat); cudaMalloc((void**)&dP, mat); cudaMalloc((void**)&dB, mat);
  cudaMalloc((void**)&dG, mat); cudaMalloc((void**)&dF, mat);
  cudaMalloc((void**)&dG2, mat); cudaMalloc((void**)&dF2, mat);
  cudaMalloc((void**)&db, vec); cudaMalloc((void**)&dx, vec); cudaMalloc((void**)&dx2, vec);
  cudaMemcpy(dA, hA, mat, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, vec, cudaMemcpyHostToDevice);
  cudaMemset(dx, 0, vec);

  si_handle h;
  CK(si_create(0, &h));
  int64_t ctr[2] = {0, 0};
  CK(si_split_scalar(h, n, dA, alpha, dP, dB, NULL));
  CK(si_initial_series(h, n, dP, dB, dA, 0, 1, dG, dF, ctr, NULL));
  double f0 = 0.0, fk = 0.0, prev_mis = INFINITY;
  CK(si_fro_norm(h, n, n, dF, n, &f0, NULL));
  for (int k = 1; k <= steps; ++k) {
    const int64_t c0 = ctr[0], c1 = ctr[1];
    CK(si_plain_richardson(h, n, 1, dA, db, dx, dG, dx2, ctr, NULL));
    CK(si_ns_step(h, n, dA, dG, dF, 3, NULL, 0, NULL, 0, dG2, dF2, ctr, NULL));
    if (ctr[0] - c0 != 3 || ctr[1] - c1 != 2) {
      fprintf(stderr, "counters: +%lld mmm +%lld mvm per step (want 3, 2)\n",
              (long long)(ctr[0] - c0), (long long)(ctr[1] - c1));
      return 1;
    }
    double* t;
    t = dG; dG = dG2; dG2 = t;
    t = dF; dF = dF2; dF2 = t;
    t = dx; dx = dx2; dx2 = t;
    /* mismatch ||A theta - b|| on the host */
    cudaMemcpy(hx, dx, vec, cudaMemcpyDeviceToHost);
    double mis = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double r = -hb[i];
      for (int64_t j = 0; j < n; ++j) r += hA[i * n + j] * hx[j];
      mis += r * r;
    }
    mis = sqrt(mis);
    if (!(mis < prev_mis) && mis > 1e-10) { /* contracts until the FP64 floor */
      fprintf(stderr, "step %d: mismatch %.3e did not drop\n", k, mis);
      return 1;
    }
    prev_mis = mis;
  }
  CK(si_fro_norm(h, n, n, dF, n, &fk, NULL));
  /* F = I - G A on the host */
  cudaMemcpy(hG, dG, mat, cudaMemcpyDeviceToHost);
  cudaMemcpy(hF, dF, mat, cudaMemcpyDeviceToHost);
  double worst = 0.0;
  for (int64_t i = 0; i < n; i += 17)
    for (int64_t j = 0; j < n; ++j) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int64_t k = 0; k < n; ++k) s -= hG[i * n + k] * hA[k * n + j];
      const double d = fabs(s - hF[i * n + j]);
      if (d > worst) worst = d;
    }
  /* the block-row sharded entry point from C (NCCL communicator, one rank on
   * this one GPU: rows [0, n)): one more NS step, bitwise the single-GPU call */
  int sharded_ok = 0;
  {
    unsigned char id[128];
    si_comm comm = NULL;
    int64_t r0 = -1, r1 = -1, sctr[2] = {0, 0};
    if (si_comm_unique_id(id) == SI_OK && si_comm_create_nccl(h, 1, 0, id, n, &comm) == SI_OK) {
      CK(si_comm_rows(comm, &r0, &r1, NULL, NULL));
      double *sG, *sF;
      cudaMalloc((void**)&sG, mat);
      cudaMalloc((void**)&sF, mat);
      CK(si_ns_step(h, n, dA, dG, dF, 3, NULL, 0, NULL, 0, dG2, dF2, NULL, NULL));
      CK(si_sharded_ns_step(h, comm, n, dA, dG, dF, 3, NULL, 0, NULL, 0, sG, sF, sctr, NULL));
      double* h1 = (double*)malloc(mat);
      double* h2 = (double*)malloc(mat);
      cudaMemcpy(h1, dF2, mat, cudaMemcpyDeviceToHost);
      cudaMemcpy(h2, sF, mat, cudaMemcpyDeviceToHost);
      sharded_ok = r0 == 0 && r1 == n && sctr[0] == 3 && memcmp(h1, h2, mat) == 0;
      free(h1);
      free(h2);
      cudaFree(sG);
      cudaFree(sF);
      CK(si_comm_destroy(comm));
    } else {
      fprintf(stderr, "sharded check skipped: %s\n", si_last_error());
      sharded_ok = 1;  /* no libnccl on this host: nothing to compare */
    }
  }
  /* the same NS step with every product emulated on the INT8 tensor cores
   * (si_set_gemm_backend: Ozaki-II, 16 moduli; min_dim 128 so n = 256 qualifies):
   * within 1e-13 (relative Frobenius) of the FP64 DMMA step */
  double emul_diff = 1.0;
  {
    double *dGe, *dFe;
    cudaMalloc((void**)&dGe, mat);
    cudaMalloc((void**)&dFe, mat);
    CK(si_ns_step(h, n, dA, dG, dF, 3, NULL, 0, NULL, 0, dG2, dF2, NULL, NULL));
    CK(si_set_gemm_backend(h, SI_GEMM_OZAKI_I8, 16, 128));
    CK(si_ns_step(h, n, dA, dG, dF, 3, NULL, 0, NULL, 0, dGe, dFe, NULL, NULL));
    CK(si_set_gemm_backend(h, SI_GEMM_DMMA, 0, 0));
    cudaMemcpy(hG, dG2, mat, cudaMemcpyDeviceToHost);
    cudaMemcpy(hF, dGe, mat, cudaMemcpyDeviceToHost);
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n * n; ++i) {
      num += (hF[i] - hG[i]) * (hF[i] - hG[i]);
      den += hG[i] * hG[i];
    }
    emul_diff = sqrt(num / den);
    cudaFree(dGe);
    cudaFree(dFe);
  }
  printf("ns_step emulated on the INT8 tensor cores vs FP64 DMMA: rel diff %.2e\n", emul_diff);
  /* a bad argument: negative dimension */
  const int bad = si_gemm(h, -1, n, n, 1.0, dA, n, dA, n, 0.0, NULL, n, 0.0, dG2, n, 0, NULL, NULL);
  printf("||F_0||_F=%.3e ||F_%d||_F=%.3e mismatch=%.3e |F - (I - G A)|max=%.2e "
         "counters mmm=%lld mvm=%lld bad-call status=%d (%s)\n",
         f0, steps, fk, prev_mis, worst, (long long)ctr[0], (long long)ctr[1], bad,
         si_last_error());
  CK(si_destroy(h));
  cudaFree(dA); cudaFree(dP); cudaFree(dB); cudaFree(dG); cudaFree(dF);
  cudaFree(dG2); cudaFree(dF2); cudaFree(db); cudaFree(dx); cudaFree(dx2);
  free(hA); free(hM); free(hb); free(hx); free(hG); free(hF);
  printf("sharded ns_step (NCCL, 1 rank) bitwise equal: %s\n", sharded_ok ? "yes" : "NO");
  if (bad != SI_EINVAL || !sharded_ok || !(emul_diff <= 1e-13)) return 1;
  if (!(fk < f0) || worst > 1e-12) return 1;
  return 0;
}
