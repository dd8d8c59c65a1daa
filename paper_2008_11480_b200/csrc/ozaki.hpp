// FP64 products emulated on the INT8 tensor cores (Ozaki scheme II): see ozaki.cu.
#pragma once
#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace si {
namespace oz {

constexpr int kMaxModuli = 16;
constexpr int kMinModuli = 8;
constexpr int kDefaultModuli = 16;
constexpr int64_t kMaxK = 65536;  // |sum of K products of int8 residues| < 2^30

// Device workspace of one emulated product, carved by the caller (engine.cu)
// from one allocation of workspace_bytes().
struct Work {
  uint8_t* base = nullptr;
  size_t bytes = 0;
};

// Bytes of device workspace an M x K by K x N product with `nmod` moduli needs.
size_t workspace_bytes(int64_t M, int64_t N, int64_t K, int nmod);

// D = alpha * (A @ B) + beta * C + diag * I (diag at (i, i + doff)), A @ B
// computed exactly from integer images of A and B on the INT8 tensor cores
// (tcgen05.mma kind::i8, one GEMM per modulus) and reconstructed by the
// Chinese remainder theorem.  Stream-ordered, no host synchronisation.
// Returns the number of kernels launched through *launches.
// ev0 / ev1 (optional) are recorded around the tensor-core kernel.
cudaError_t launch_gemm(const Mat& A, const Mat& B, Mat& D, const Epilogue& e, int nmod,
                        const Work& w, cudaStream_t s, int64_t* launches,
                        cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr);

// Test hook for the tensor-core kernel alone: R[l] = (A[l] @ Bt[l]^T) mod m_l
// for l < nplanes, A[l]: M x Kp int8 rows, Bt[l]: N x Kp int8 rows (K-major,
// Kp a multiple of 128, columns >= K zero), R[l]: M x N uint8.
cudaError_t launch_i8_gemm_mod(const int8_t* A, const int8_t* Bt, uint8_t* R, int64_t M, int64_t N,
                               int64_t Kp, int nplanes, cudaStream_t s);

// Moduli (pairwise coprime, <= 256) in the order the planes use them.
unsigned modulus(int l);

}  // namespace oz
}  // namespace si
