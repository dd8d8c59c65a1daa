// FP64 products emulated on the INT8 tensor cores (Ozaki scheme II): see ozaki.cu.
#pragma once
#include <cstddef>
#include <cstdint>
#include <functional>

#include "common.cuh"

namespace si {
namespace oz {

constexpr int kMaxModuli = 16;
constexpr int kMinModuli = 8;
constexpr int kDefaultModuli = 16;
constexpr int64_t kMaxK = 65536;  // |sum of K products of int8 residues| < 2^30

// Device workspace of one emulated product, carved by the caller (engine.cu)
// from one allocation of workspace_bytes().
// INT8 tensor-core kernel: single CTAs (cta_group::1, 128 x 256 tiles; the
// default) or CTA pairs (cta_group::2, 256 x 256 tiles: more work per clock,
// but twice the DRAM bytes, which costs more at the 1000 W cap -- 10% slower
// in the C4 step, profiles/ozaki_kernel_ab_r02.txt).  Identical results.
constexpr int kI8Auto = 0, kI8Pair = 1, kI8Single = 2;
// single-CTA MMAs on 2-CTA clusters sharing (multicasting) the B tile
constexpr int kI8Multicast = 3;

struct Work {
  uint8_t* base = nullptr;
  size_t bytes = 0;
  int64_t max_cols = 0;  // columns of D per chunk at most (0: kChunkBudget decides)
  int64_t max_rows = 0;  // rows of D per chunk at most (0: all rows)
  int variant = kI8Auto;  // INT8 kernel
};

// Column chunking: the B-side residue planes and the result planes of one
// chunk of D's columns take at most this many bytes (the A-side planes are
// built once and shared by every chunk), so a 32768^2 product needs ~28 GB
// of workspace instead of ~52 GB.
constexpr size_t kChunkBudget = (size_t)10 << 30;

// Bytes of device workspace an M x K by K x N product with `nmod` moduli needs.
// `max_rows`, `max_cols` as in Work.  With several row chunks the B-side
// planes are rebuilt per row chunk (unless one column chunk covers N).
size_t workspace_bytes(int64_t M, int64_t N, int64_t K, int nmod, int64_t max_cols = 0,
                       int64_t max_rows = 0);

// Scales + residue planes of one operand side, kept by the caller across
// products that share the operand (engine.cu: a step's immutable inputs).
// `ready` = already filled (stream-ordered before this launch); otherwise
// launch_gemm fills them.  Used only when the product is not chunked on that
// side (rows of A / columns of B).
struct Side {
  unsigned long long* scale = nullptr;  // max |entry| bits per row (A) / column (B)
  int8_t* planes = nullptr;             // nmod x rows x Kp (A) / nmod x cols x Kp (B)
  bool ready = false;
};
size_t side_bytes(int64_t rows, int64_t K, int nmod);  // scale + planes, 256-aligned parts

// Called on the stream right before (begin = true) and after (false) every
// INT8 tensor-core launch of a product, with that launch's int8 op count
// (2 M Nc Kp per plane, summed over planes) -- the profiling hook.
using I8Hook = std::function<void(bool begin, double ops)>;

// Called on the stream before the A-side work of each row chunk [r0, r1) of D
// (e.g. waits for the rows of A still being copied in).
using RowHook = std::function<void(int64_t r0, int64_t r1)>;

// D = alpha * (A @ B) + beta * C + diag * I (diag at (i, i + doff)), A @ B
// computed exactly from integer images of A and B on the INT8 tensor cores
// (tcgen05.mma kind::i8, one GEMM per modulus) and reconstructed by the
// Chinese remainder theorem.  Stream-ordered, no host synchronisation.
// Returns the number of kernels launched through *launches.
cudaError_t launch_gemm(const Mat& A, const Mat& B, Mat& D, const Epilogue& e, int nmod,
                        const Work& w, cudaStream_t s, int64_t* launches,
                        const I8Hook& hook = nullptr, Side* a_side = nullptr,
                        Side* b_side = nullptr, const RowHook& row_hook = nullptr);

// Sum-of-squares slots launch_gemm writes when e.sq is set (D's ||.||_F^2 =
// the fixed-order sum of these; one slot per warp of each CRT launch).
int64_t sq_slots(int64_t M, int64_t N, int64_t K, int nmod, const Work& w);

// Test hook for the tensor-core kernel alone: R[l] = (A[l] @ Bt[l]^T) mod m_l
// for l < nplanes, A[l]: M x Kp int8 rows, Bt[l]: N x Kp int8 rows (K-major,
// Kp a multiple of 128, columns >= K zero), R[l]: M x N uint8.
cudaError_t launch_i8_gemm_mod(const int8_t* A, const int8_t* Bt, uint8_t* R, int64_t M, int64_t N,
                               int64_t Kp, int nplanes, cudaStream_t s, int variant = kI8Auto);

// Tuning hook of the INT8 kernels (process-wide): rasterisation group
// (pair-tile rows per group) and the L2 policies of the A / B operand loads
// (0 evict_normal, 1 evict_last, 2 evict_first); negative / zero keeps a value.
void tune_pair(int group_m, int l2a, int l2b);
void tune_pair_stages(int stages);
// Longest K range one launch of the single-CTA kernel covers (longer products
// run as several launches accumulating residues in R; 0 = never split, the
// default).
void tune_ksplit(int64_t kmax);

// Moduli (pairwise coprime, <= 256) in the order the planes use them.
unsigned modulus(int l);

}  // namespace oz
}  // namespace si
