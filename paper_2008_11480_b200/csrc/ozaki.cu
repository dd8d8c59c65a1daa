// FP64 products emulated on the INT8 tensor cores of sm_100a (Ozaki scheme II).
//
// FP64 tensor work on B200 runs on the warp-level DMMA pipe (37 TFLOP/s,
// gemm_tma.cu): tcgen05.mma has no f64 kind.  It does have kind::i8 (int8 x
// int8 -> int32 in TMEM) at 4.5 POPS dense, and an FP64 product can be computed
// EXACTLY from integers:
//
//  1. Scale (per row of A, per column of B, by powers of two) and round to
//     integers: A' = rint(diag(2^sa) A), B' = rint(B diag(2^sb)), with
//     |A'| <= 2^pa, |B'| <= 2^pb and K * 2^(pa+pb) <= M/4, M = prod m_l.
//     Only this rounding loses information: every entry keeps the bits of its
//     row's (column's) largest entry down to 2^-pa relative, pa, pb ~ 54 for
//     16 moduli at K = 16384 -- as fine as the 53-bit significand of the
//     largest entries themselves.
//  2. For each modulus m_l (pairwise coprime, <= 256): residues of A' and B'
//     in [-128, 127] (int8), and C_l = A'_l @ B'_l on the tensor cores.  The
//     int32 sums are exact (|C_l| <= K * 2^14 <= 2^30 for K <= 65536), reduced
//     mod m_l in the TMEM epilogue and stored as one byte per entry.
//  3. C' = A' B' is the unique integer in (-M/4, M/4] with those residues
//     (Chinese remainder theorem), rebuilt in FP64 from exact partial sums
//     (32-bit pieces of the CRT weights) and scaled back by 2^-(sa_i + sb_j);
//     the seriesinv epilogue (alpha, beta * C, diag * I) is fused there.
//
// The integer product is exact and order-free, so results do not depend on
// tiling, chunking, concurrency or on how rows are split across ranks (the
// block-row sharded path stays bitwise equal to the single-GPU call, as with
// DMMA).
//
// Kernels (one emulated product = 6 launches per row x column chunk):
//   row_absmax / col_absmax      max |a| per row of A, per column of B (HBM)
//   residues_rows / residues_cols A -> nmod int8 planes (K-major), B -> nmod
//                                int8 planes transposed to K-major (INT pipe)
//   i8_gemm_mod_kernel           nmod int8 GEMMs, tcgen05.mma kind::i8 with
//                                TMA (128B swizzle) -> 4-stage smem ring ->
//                                single-thread MMA issue -> double-buffered
//                                TMEM accumulators -> 4 epilogue warps
//                                (tcgen05.ld, mod m_l, byte stores); the
//                                default.  Variants: i8_gemm_mod_pair_kernel
//                                (cta_group::2 CTA pairs) and
//                                i8_gemm_mod_mc_kernel (B tiles multicast in
//                                2-CTA clusters), measured and kept selectable
//   crt_kernel<NMOD>             CRT + scale + fused epilogue (FP64 pipe)
// The scales + residue planes of a step's immutable operands are kept across
// the step's products by the caller (engine.cu, `Side`).
#include "ozaki.hpp"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstring>
#include <mutex>

namespace si {
namespace oz {
namespace {

// ---------------------------------------------------------------- moduli --
__host__ __device__ constexpr unsigned kmod(int l) {
  return l == 0    ? 256u
         : l == 1  ? 255u
         : l == 2  ? 253u
         : l == 3  ? 251u
         : l == 4  ? 247u
         : l == 5  ? 241u
         : l == 6  ? 239u
         : l == 7  ? 233u
         : l == 8  ? 229u
         : l == 9  ? 227u
         : l == 10 ? 223u
         : l == 11 ? 217u
         : l == 12 ? 211u
         : l == 13 ? 199u
         : l == 14 ? 197u
                   : 193u;
}
__host__ __device__ constexpr unsigned pow2mod(int e, unsigned m) {
  unsigned r = 1u % m;
  for (int i = 0; i < e; ++i) r = (r * 2u) % m;
  return r;
}

constexpr int kNonFinite = INT_MIN / 4;  // shift sentinel: the row / column holds inf or nan
constexpr unsigned long long kInfBits = 0x7FF0000000000000ull;
constexpr int kMaxP = 56;  // |A'| <= 2^56 keeps u = A' + 2^57 below 2^58

__device__ __forceinline__ int shift_of(unsigned long long maxbits, int p) {
  if (maxbits >= kInfBits) return kNonFinite;
  if (maxbits == 0ull) return 0;
  return p - 1 - ilogb(__longlong_as_double((long long)maxbits));
}

// a * 2^sh (exact while the result is >= 2^-1022 or rounds to 0 under rint)
__device__ __forceinline__ double pow2(int e) {  // -1022 <= e <= 1023
  return __longlong_as_double((long long)(e + 1023) << 52);
}

// Symmetric residue modulo kmod(L) of the integer x = u - 2^57, u < 2^58 given
// as 20-bit chunks u = c2 2^40 + c1 2^20 + c0: one reduction of
// c2 (2^40 mod m) + c1 (2^20 mod m) + c0 + (m - 2^57 mod m) < 2^29, then the
// symmetric representative in [-(m-1)/2, m/2) -- int8 for every modulus <= 256.
struct Chunks {
  uint32_t c0, c1, c2;
};
__device__ __forceinline__ Chunks chunks_of(long long x) {
  const unsigned long long u = (unsigned long long)(x + (1ll << 57));
  return Chunks{(uint32_t)u & 0xFFFFFu, (uint32_t)(u >> 20) & 0xFFFFFu, (uint32_t)(u >> 40)};
}
// (x + h) mod m with h = m / 2, i.e. the symmetric residue plus h, in [0, m)
template <int L>
__device__ __forceinline__ uint32_t res_shifted(const Chunks& c) {
  constexpr unsigned m = kmod(L);
  constexpr unsigned r40 = pow2mod(40, m);
  constexpr unsigned r20 = pow2mod(20, m);
  constexpr unsigned kh = (m - pow2mod(57, m) + m / 2) % m;
  return (c.c2 * r40 + c.c1 * r20 + c.c0 + kh) % m;
}

// four shifted residues r_j in [0, m) -> one word of the int8 values r_j - h
// (two's complement bytes): byte packing by PRMT, then a carry-free per-byte
// subtraction of h
template <int L>
__device__ __forceinline__ uint32_t pack_sym4(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  constexpr unsigned h = kmod(L) / 2;
  const uint32_t w = __byte_perm(__byte_perm(r0, r1, 0x0040), __byte_perm(r2, r3, 0x0040), 0x5410);
  constexpr uint32_t H = (uint32_t)((256u - h) & 0xFFu) * 0x01010101u;  // + (256 - h) per byte
  return ((w & 0x7F7F7F7Fu) + (H & 0x7F7F7F7Fu)) ^ ((w ^ H) & 0x80808080u);
}

// integer image rint(a * 2^sh) of a (sh not the sentinel)
__device__ __forceinline__ long long int_image(double a, int sh) {
  if (sh > 1000) {
    a *= pow2(600);
    sh -= 600;
  }
  return __double2ll_rn(a * pow2(sh));
}


// ------------------------------------------------------------- scaling --
// max |a_ij| over each row (as the bit pattern of |a|: ordered like the value,
// inf / nan above every finite value); one warp per row.
__global__ void row_absmax_kernel(const double* __restrict__ A, int64_t lda, int M, int K,
                                  unsigned long long* __restrict__ out) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < M; row += warps) {
    const double* p = A + (int64_t)row * lda;
    unsigned long long m = 0ull;
    int k = lane;
    for (; k + 96 < K; k += 128) {
      const double v0 = p[k], v1 = p[k + 32], v2 = p[k + 64], v3 = p[k + 96];
      m = max(m, (unsigned long long)__double_as_longlong(fabs(v0)));
      m = max(m, (unsigned long long)__double_as_longlong(fabs(v1)));
      m = max(m, (unsigned long long)__double_as_longlong(fabs(v2)));
      m = max(m, (unsigned long long)__double_as_longlong(fabs(v3)));
    }
    for (; k < K; k += 32) m = max(m, (unsigned long long)__double_as_longlong(fabs(p[k])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) out[row] = m;
  }
}

// max |b_ij| over each column: 32 columns x 256 rows per block, atomicMax into
// `out` (zeroed by the caller).
__global__ void col_absmax_kernel(const double* __restrict__ B, int64_t ldb, int K, int N,
                                  unsigned long long* __restrict__ out) {
  __shared__ unsigned long long red[8][32];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  const int k0 = blockIdx.y * 256;
  unsigned long long m = 0ull;
  if (j < N) {
    const int k1 = min(K, k0 + 256);
    for (int k = k0 + ty; k < k1; k += 8)
      m = max(m, (unsigned long long)__double_as_longlong(fabs(B[(int64_t)k * ldb + j])));
  }
  red[ty][tx] = m;
  __syncthreads();
  if (ty == 0 && j < N) {
#pragma unroll
    for (int i = 1; i < 8; ++i) m = max(m, red[i][tx]);
    if (m) atomicMax(out + j, m);
  }
}

// ------------------------------------------------------------ residues --
// residues of 16 consecutive integers modulo kmod(L), kmod(L+1), ... (L < nmod),
// one 16-byte store into each plane
template <int L, int E>
__device__ __forceinline__ void emit(int nmod, const Chunks (&x)[E], int8_t* dst, int64_t plane) {
  static_assert(E == 8 || E == 16, "8 or 16 residues per store");
  if constexpr (L < kMaxModuli) {
    if (L >= nmod) return;
    uint32_t r[E];
#pragma unroll
    for (int j = 0; j < E; ++j) r[j] = res_shifted<L>(x[j]);
    if constexpr (E == 16) {
      uint4 w;
      w.x = pack_sym4<L>(r[0], r[1], r[2], r[3]);
      w.y = pack_sym4<L>(r[4], r[5], r[6], r[7]);
      w.z = pack_sym4<L>(r[8], r[9], r[10], r[11]);
      w.w = pack_sym4<L>(r[12], r[13], r[14], r[15]);
      *reinterpret_cast<uint4*>(dst + L * plane) = w;
    } else {
      uint2 w;
      w.x = pack_sym4<L>(r[0], r[1], r[2], r[3]);
      w.y = pack_sym4<L>(r[4], r[5], r[6], r[7]);
      *reinterpret_cast<uint2*>(dst + L * plane) = w;
    }
    emit<L + 1, E>(nmod, x, dst, plane);
  }
}

// A (M x K, row-major) -> nmod planes of M x Kp int8 (columns >= K zero):
// one thread per RE consecutive k of a row, one RE-byte store per plane (8:
// fewer registers per thread, twice the resident warps of 16)
constexpr int RE = 8;
__global__ void residues_rows_kernel(const double* __restrict__ A, int64_t lda, int M, int K,
                                     int Kp, const unsigned long long* __restrict__ rmax, int p,
                                     int nmod, int8_t* __restrict__ out) {
  const int chunks = Kp / RE;
  const int64_t total = (int64_t)M * chunks;
  const int64_t plane = (int64_t)M * Kp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx / chunks);
    const int k0 = (int)(idx - (int64_t)row * chunks) * RE;
    const int sh = shift_of(rmax[row], p);
    Chunks x[RE];
    const double* src = A + (int64_t)row * lda + k0;
    if (sh == kNonFinite) {
#pragma unroll
      for (int j = 0; j < RE; ++j) x[j] = chunks_of(0);
    } else if (k0 + RE <= K && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0)) {
#pragma unroll
      for (int j = 0; j < RE; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(src + j);
        x[j] = chunks_of(int_image(v.x, sh));
        x[j + 1] = chunks_of(int_image(v.y, sh));
      }
    } else {
#pragma unroll
      for (int j = 0; j < RE; ++j) x[j] = chunks_of(k0 + j < K ? int_image(src[j], sh) : 0);
    }
    emit<0, RE>(nmod, x, out + (int64_t)row * Kp + k0, plane);
  }
}

// B (K x N, row-major) -> nmod planes of N x Kp int8, transposed (row j of a
// plane = column j of B, K contiguous): 64 k x 64 j tiles through shared memory.
__global__ void __launch_bounds__(256) residues_cols_kernel(
    const double* __restrict__ B, int64_t ldb, int K, int N, int Kp,
    const unsigned long long* __restrict__ cmax, int p, int nmod, int8_t* __restrict__ out) {
  __shared__ long long xs[64][65];
  __shared__ int shs[64];
  const int k0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tid = threadIdx.x;
  if (tid < 64) shs[tid] = (j0 + tid < N) ? shift_of(cmax[j0 + tid], p) : 0;
  __syncthreads();
  {
    const int tx = tid & 63, ty = tid >> 6;
    const int j = j0 + tx;
    const int sh = shs[tx];
#pragma unroll 4
    for (int r = ty; r < 64; r += 4) {
      const int k = k0 + r;
      const long long x = (j < N && k < K && sh != kNonFinite) ? int_image(B[(int64_t)k * ldb + j], sh) : 0;
      xs[r][tx] = x;
    }
  }
  __syncthreads();
  const int jl = tid >> 2, kc = (tid & 3) << 4;
  if (j0 + jl >= N || k0 + kc >= Kp) return;
  Chunks x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = chunks_of(xs[kc + i][jl]);
  emit<0, 16>(nmod, x, out + (int64_t)(j0 + jl) * Kp + k0 + kc, (int64_t)N * Kp);
}

// -------------------------------------------------- INT8 tensor-core GEMM --
constexpr int GBM = 128, GBN = 256, GBK = 128;  // CTA tile; GBK in bytes (= int8 elements)
constexpr int GSTAGES = 4;
constexpr int GA_BYTES = GBM * GBK;  // 16 KB
constexpr int GB_BYTES = GBN * GBK;  // 32 KB
constexpr int GSTAGE_BYTES = GA_BYTES + GB_BYTES;
constexpr int GTHREADS = 192;  // warp 0 TMA, warp 1 MMA + TMEM owner, warps 2-5 epilogue
constexpr int GSMEM = GSTAGES * GSTAGE_BYTES + 1024 + 256;
constexpr int GROUP_M = 16;
constexpr int kTmemCols = 2 * GBN;  // two 128 x 256 int32 accumulators (all of TMEM)
// instruction descriptor, kind::i8: D s32 [4,6), A s8 [7,10), B s8 [10,13),
// both K-major, N >> 3 at [17,23), M >> 4 at [24,29)
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(GBN >> 3) << 17) |
                            ((uint32_t)(GBM >> 4) << 24);

// per-plane reduction of the int32 sums: r = v mod m from u = v + 2^30 < 2^31,
// q = floor(u * magic / 2^39) with magic = floor(2^39 / m) + 1 (exact for u < 2^31)
struct ModTab {
  unsigned m[kMaxModuli];
  unsigned magic[kMaxModuli];
  unsigned off[kMaxModuli];  // 2^30 mod m
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// shared-memory matrix descriptor: K-major, 128B swizzle (8-row groups 1024 B
// apart), sm_100 version bits
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}


// Epilogue of one accumulator: this thread's TMEM lane holds row `row` of a
// 256-column tile (from column `taddr`); the int32 sums are reduced exactly
// mod m (u = v + 2^30 < 2^31, q = floor(u magic / 2^39)) and stored as one
// byte per entry into row `row`, columns col0.. of the plane.
// `accum`: the plane already holds the residues of an earlier K range of the
// same product (launch_i8_gemm_mod's K split); they are added before the
// reduction (|v| <= 2^29 per range, + 255: still below 2^31 after the shift).
// (a template parameter: the default instantiation is the plain epilogue, and
// every index into v[] stays a compile-time constant -- a dynamically indexed
// v[] would live in local memory and slow the epilogue of every launch)
template <bool ACCUM = false>
__device__ __forceinline__ void store_mod_row(uint32_t taddr, uint8_t* __restrict__ plane_base,
                                              int row, int col0, int M, int N, unsigned m,
                                              unsigned magic, unsigned off) {
  uint8_t* rp = plane_base + (int64_t)row * N + col0;
  const bool vec = ((N & 15) == 0);
#pragma unroll 1
  for (int c = 0; c < 256 / 32; ++c) {
    uint32_t v[32];
    tmem_ld32(taddr + (uint32_t)(c * 32), v);
    if constexpr (ACCUM) {
      if (row < M && col0 + c * 32 < N) {
        if (vec && col0 + c * 32 + 32 <= N) {
          const uint4* src = reinterpret_cast<const uint4*>(rp + c * 32);
          const uint4 p0 = src[0], p1 = src[1];
          const uint32_t pw[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += (pw[i >> 2] >> (8 * (i & 3))) & 0xFFu;
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (col0 + c * 32 + i < N) v[i] += rp[c * 32 + i];
        }
      }
    }
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      uint32_t b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t u = v[i + j] + (1u << 30);
        const uint32_t qq = __umulhi(u, magic) >> 7;
        uint32_t r = u - qq * m;
        r = r >= off ? r - off : r + m - off;
        b[j] = r;
      }
      w[i >> 2] = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
    }
    const int cc = col0 + c * 32;
    if (row < M && cc < N) {
      if (vec && cc + 32 <= N) {
        uint4* dst = reinterpret_cast<uint4*>(rp + c * 32);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      } else {
        for (int i = 0; i < 32 && cc + i < N; ++i) rp[c * 32 + i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
      }
    }
  }
}

__device__ __forceinline__ void tile_of(int t, int num_m, int num_n, int& plane, int& tm, int& tn,
                                        int group_m = GROUP_M) {
  const int per_plane = num_m * num_n;
  plane = t / per_plane;
  const int r = t - plane * per_plane;
  const int per_group = group_m * num_n;
  const int group = r / per_group;
  const int first_m = group * group_m;
  const int gsize = min(num_m - first_m, group_m);
  const int q = r - group * per_group;
  tm = first_m + q % gsize;
  tn = q / gsize;
}

// R[l] = (A[l] @ Bt[l]^T) mod m_l, persistent over (plane, row tile, column tile)
template <bool ACCUM>
__global__ void __launch_bounds__(GTHREADS, 1)
    i8_gemm_mod_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, uint8_t* R, int M,
                       int N, int kb0, int kblocks, int nplanes,
                       const __grid_constant__ ModTab mt, int group_m) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + GSTAGES * GSTAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (GSTAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * GSTAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * GSTAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * GSTAGES + 4);
  uint8_t* smem_gen = smem_raw + (tmem_slot - raw);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (M + GBM - 1) / GBM;
  const int num_n = (N + GBN - 1) / GBN;
  const int total = num_m * num_n * nplanes;  // k-blocks [kb0, kb0 + kblocks) of every tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tmem_slot),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(smem_gen);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int plane, tm, tn;
        tile_of(t, num_m, num_n, plane, tm, tn, group_m);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          const uint32_t sa = base + stage * GSTAGE_BYTES;
          mbar_expect_tx(full_bar(stage), GSTAGE_BYTES);
          tma_load_3d(sa, &tmA, full_bar(stage), (kb0 + kb) * GBK, tm * GBM, plane);
          tma_load_3d(sa + GA_BYTES, &tmB, full_bar(stage), (kb0 + kb) * GBK, tn * GBN, plane);
          if (++stage == GSTAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (one thread) ----------------
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(tempty_bar(acc), aphase ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * GBN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t sa = base + stage * GSTAGE_BYTES;
          const uint64_t adesc = sdesc(sa), bdesc = sdesc(sa + GA_BYTES);
#pragma unroll
          for (int k = 0; k < GBK / 32; ++k)  // K = 32 bytes per MMA: +2 in the 16-byte address field
            mma_i8(d, adesc + 2 * k, bdesc + 2 * k, (kb | k) != 0 ? 1u : 0u);
          mma_commit(empty_bar(stage));  // frees the stage once these MMAs have read it
          if (++stage == GSTAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit(tfull_bar(acc));  // accumulator complete
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1u;
        }
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> mod m_l -> bytes ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int plane, tm, tn;
      tile_of(t, num_m, num_n, plane, tm, tn, group_m);
      const unsigned m = mt.m[plane], magic = mt.magic[plane], off = mt.off[plane];
      mbar_wait(tfull_bar(acc), aphase);
      tc_fence_after();
      const int row = tm * GBM + q * 32 + lane;
      const int col0 = tn * GBN;
      store_mod_row<ACCUM>(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * GBN),
                           R + (int64_t)plane * M * N, row, col0, M, N, m, magic, off);
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// ---------------------------------------- INT8 GEMM on CTA pairs (2 SMs) --
// Same product as i8_gemm_mod_kernel on 256 x 256 pair tiles: a 2-CTA cluster
// issues tcgen05.mma.cta_group::2 (M = 256, N = 256) from the leader CTA; each
// CTA stages its own 128 rows of A and 128 of the 256 rows of Bt (half of the
// B tile), so per SM the shared-memory operand traffic per MMA is 8 KB instead
// of 12 KB for the single-CTA 128 x 256 tile, and every Bt / A k-slab crosses
// L2 once per pair.  TMA of both CTAs completes on the leader's full barrier;
// the leader's MMA commits free the stage in both CTAs (multicast); each CTA's
// epilogue drains its own TMEM rows and arrives on the leader's TMEM-empty
// barrier.
constexpr int PBM = 256, PBN = 256;  // pair tile (each CTA: 128 rows of A, 128 rows of Bt)
constexpr int PA_BYTES = (PBM / 2) * GBK;  // 16 KB
constexpr int PB_BYTES = (PBN / 2) * GBK;  // 16 KB
constexpr int PSTAGE_BYTES = PA_BYTES + PB_BYTES;
constexpr int psmem(int stages) { return stages * PSTAGE_BYTES + 1024 + 256; }
constexpr uint32_t kIdescPair = (2u << 4) | (1u << 7) | (1u << 10) |
                                ((uint32_t)(PBN >> 3) << 17) | ((uint32_t)(PBM >> 4) << 24);

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t leader_addr(uint32_t a) {  // a in the leader CTA's window
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int c0, int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}
// L2 policies of the operand loads: 0 evict_normal, 1 evict_last, 2 evict_first
__device__ __forceinline__ uint64_t l2_policy(int kind) {
  uint64_t p;
  if (kind == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 2)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescPair), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {  // both CTAs' barrier at `bar`
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}

template <int PSTAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GTHREADS, 1)
    i8_gemm_mod_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                            const __grid_constant__ CUtensorMap tmB, uint8_t* __restrict__ R,
                            int M, int N, int Kp, int nplanes, const __grid_constant__ ModTab mt,
                            int group_m, int l2a, int l2b) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + PSTAGES * PSTAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (PSTAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * PSTAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * PSTAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * PSTAGES + 4);
  uint8_t* smem_gen = smem_raw + (tmem_slot - raw);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int num_m = (M + PBM - 1) / PBM;
  const int num_n = (N + PBN - 1) / PBN;
  const int total = num_m * num_n * nplanes;
  const int kblocks = Kp / GBK;
  const int cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 2 * 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tmem_slot),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(smem_gen);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs: own A rows, own half of Bt) ----
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      const uint64_t pol_a = l2_policy(l2a), pol_b = l2_policy(l2b);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < total; t += nclusters) {
        int plane, tm, tn;
        tile_of(t, num_m, num_n, plane, tm, tn, group_m);
        const int arow = tm * PBM + (int)rank * (PBM / 2);
        const int brow = tn * PBN + (int)rank * (PBN / 2);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          const uint32_t sa = base + stage * PSTAGE_BYTES;
          const uint32_t fb = leader_addr(full_bar(stage));
          if (rank == 0) mbar_expect_tx(full_bar(stage), 2 * PSTAGE_BYTES);
          tma_load_3d_pair(sa, &tmA, fb, kb * GBK, arow, plane, pol_a);
          tma_load_3d_pair(sa + PA_BYTES, &tmB, fb, kb * GBK, brow, plane, pol_b);
          if (++stage == PSTAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader CTA, one thread) ----------------
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int t = cid; t < total; t += nclusters) {
        mbar_wait(tempty_bar(acc), aphase ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * PBN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t sa = base + stage * PSTAGE_BYTES;
          const uint64_t adesc = sdesc(sa), bdesc = sdesc(sa + PA_BYTES);
#pragma unroll
          for (int k = 0; k < GBK / 32; ++k)
            mma_i8_pair(d, adesc + 2 * k, bdesc + 2 * k, (kb | k) != 0 ? 1u : 0u);
          mma_commit_pair(empty_bar(stage));
          if (++stage == PSTAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit_pair(tfull_bar(acc));
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1u;
        }
      }
    }
  } else {
    // ---------------- epilogue (both CTAs: own 128 rows of the pair tile) ----
    const int q = warp & 3;
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = cid; t < total; t += nclusters) {
      int plane, tm, tn;
      tile_of(t, num_m, num_n, plane, tm, tn, group_m);
      const unsigned m = mt.m[plane], magic = mt.magic[plane], off = mt.off[plane];
      mbar_wait(tfull_bar(acc), aphase);
      tc_fence_after();
      const int row = tm * PBM + (int)rank * (PBM / 2) + q * 32 + lane;
      const int col0 = tn * PBN;
      store_mod_row(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * PBN),
                    R + (int64_t)plane * M * N, row, col0, M, N, m, magic, off);
      tc_fence_before();
      mbar_arrive_cluster(leader_addr(tempty_bar(acc)));
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1u;
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// ------------------------------- INT8 GEMM, B tiles multicast in CTA pairs --
// Single-CTA MMAs (cta_group::1, 128 x 256 per CTA) on 2-CTA clusters whose
// CTAs take adjacent 128-row tiles of the same 256-column tile: each CTA loads
// its own A rows and HALF of the Bt tile with `.multicast::cluster`, which
// lands in both CTAs' shared memory -- per SM 32 KB of L2 reads per k-block
// instead of 48 KB, with the single-CTA kernel's accumulators and epilogue.
// A stage is refilled only when both CTAs' MMAs have read it (each MMA commit
// arrives on both CTAs' empty barrier, count 2).
__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                               int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mma_commit_both(uint32_t bar) {  // this CTA's MMAs -> both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GTHREADS, 1)
    i8_gemm_mod_mc_kernel(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmB, uint8_t* __restrict__ R, int M,
                          int N, int Kp, int nplanes, const __grid_constant__ ModTab mt,
                          int group_m) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + GSTAGES * GSTAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (GSTAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * GSTAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * GSTAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * GSTAGES + 4);
  uint8_t* smem_gen = smem_raw + (tmem_slot - raw);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = (int)cta_rank();
  const int num_m = (M + 2 * GBM - 1) / (2 * GBM);  // 256-row tile pairs
  const int num_n = (N + GBN - 1) / GBN;
  const int total = num_m * num_n * nplanes;
  const int kblocks = Kp / GBK;
  const int cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  constexpr int kHalfB = GB_BYTES / 2;  // 128 rows of Bt per CTA

  if (threadIdx.x == 0) {
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 2);  // both CTAs' MMAs
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tmem_slot),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();  // the peer's barriers are initialised before any multicast reaches them
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(smem_gen);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: own A rows, half of Bt to both CTAs ----
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < total; t += nclusters) {
        int plane, tm, tn;
        tile_of(t, num_m, num_n, plane, tm, tn, group_m);
        const int arow = tm * 2 * GBM + rank * GBM;
        const int brow = tn * GBN + rank * (GBN / 2);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1u);  // both CTAs are done with this stage
          const uint32_t sa = base + stage * GSTAGE_BYTES;
          mbar_expect_tx(full_bar(stage), GSTAGE_BYTES);
          tma_load_3d(sa, &tmA, full_bar(stage), kb * GBK, arow, plane);
          tma_load_3d_mc(sa + GA_BYTES + rank * kHalfB, &tmB, full_bar(stage), kb * GBK, brow,
                         plane);
          if (++stage == GSTAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      // drain: every commit of both CTAs' MMAs has reached this CTA's empty
      // barriers before the cluster may exit
      for (int i = 0; i < GSTAGES; ++i) {
        mbar_wait(empty_bar(stage), phase ^ 1u);
        if (++stage == GSTAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (one thread per CTA) ----------------
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int t = cid; t < total; t += nclusters) {
        mbar_wait(tempty_bar(acc), aphase ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * GBN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t sa = base + stage * GSTAGE_BYTES;
          const uint64_t adesc = sdesc(sa), bdesc = sdesc(sa + GA_BYTES);
#pragma unroll
          for (int k = 0; k < GBK / 32; ++k)
            mma_i8(d, adesc + 2 * k, bdesc + 2 * k, (kb | k) != 0 ? 1u : 0u);
          mma_commit_both(empty_bar(stage));
          if (++stage == GSTAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit(tfull_bar(acc));
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1u;
        }
      }
    }
  } else {
    // ---------------- epilogue: own 128 rows ----------------
    const int q = warp & 3;
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = cid; t < total; t += nclusters) {
      int plane, tm, tn;
      tile_of(t, num_m, num_n, plane, tm, tn, group_m);
      const unsigned m = mt.m[plane], magic = mt.magic[plane], off = mt.off[plane];
      mbar_wait(tfull_bar(acc), aphase);
      tc_fence_after();
      const int row = tm * 2 * GBM + rank * GBM + q * 32 + lane;
      const int col0 = tn * GBN;
      store_mod_row(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * GBN),
                    R + (int64_t)plane * M * N, row, col0, M, N, m, magic, off);
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1u;
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// ------------------------------------------------------------------ CRT --
// X = sum_l c_l W_l (W_l the CRT weights, c_l in [0, m_l)) is held exactly as
// four partial sums S_k of 32-bit pieces (c_l * piece < 2^40, 16 terms < 2^44);
// q = rint(X / M); C' = X - q M = sum_k (S_k - q M_k) 2^(32k), every S_k - q M_k
// exact, combined most significant first.
struct CrtTab {
  double w[kMaxModuli][4];  // pieces of W_l: w[l][k] = (W_l >> 32k) & 0xffffffff
  double mp[4];             // pieces of M
  double inv_m;             // 1 / M (rounded)
  int nmod;
};

// alpha * acc + beta * c with one rounding for the sum (alpha = +-1, beta = 1:
// the exactly rounded acc +- c)
__device__ __forceinline__ double apply_epi(double acc, double alpha, double beta, double cval) {
  const double v = __dmul_rn(alpha, acc);
  return beta != 0.0 ? __fma_rn(beta, cval, v) : v;
}

// byte j of w as a double: the bits of 2^52 + byte, minus 2^52 (one DADD on the
// FP64 pipe instead of an I2F conversion)
__device__ __forceinline__ double byte_f64(uint32_t w, int j) {
  return __hiloint2double(0x43300000, (int)((w >> (8 * j)) & 0xFFu)) - 0x1p52;
}

// the CRT sums of the 4 entries packed in w[l] (byte j = entry j), planes
// outermost so each CRT constant is loaded once per 4 entries
template <int NMOD>
__device__ __forceinline__ void crt_values4(const uint32_t (&w)[NMOD], const CrtTab& t,
                                            double (&out)[4]) {
  double sum[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) sum[j][0] = sum[j][1] = sum[j][2] = sum[j][3] = 0.0;
#pragma unroll
  for (int l = 0; l < NMOD; ++l) {
    const double w0 = t.w[l][0], w1 = t.w[l][1], w2 = t.w[l][2], w3 = t.w[l][3];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double cl = byte_f64(w[l], j);
      sum[j][0] = fma(cl, w0, sum[j][0]);
      sum[j][1] = fma(cl, w1, sum[j][1]);
      sum[j][2] = fma(cl, w2, sum[j][2]);
      sum[j][3] = fma(cl, w3, sum[j][3]);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double s0 = sum[j][0], s1 = sum[j][1], s2 = sum[j][2], s3 = sum[j][3];
    const double x = fma(s3, 0x1p96, fma(s2, 0x1p64, s1 * 0x1p32));
    const double q = rint(x * t.inv_m);
    const double t3 = fma(-q, t.mp[3], s3), t2 = fma(-q, t.mp[2], s2);
    const double t1 = fma(-q, t.mp[1], s1), t0 = fma(-q, t.mp[0], s0);
    out[j] = fma(fma(fma(t3, 0x1p32, t2), 0x1p32, t1), 0x1p32, t0);
  }
}

// v * 2^e, one rounding
__device__ __forceinline__ double scale2(double v, int e) {
  return (e >= -1022 && e <= 1023) ? v * pow2(e) : ldexp(v, e);
}

// one thread per 4 consecutive columns of a row (one 32-bit load per plane);
// the moduli count is a template parameter (no per-plane branches)
template <int NMOD>
__global__ void __launch_bounds__(256) crt_kernel(
    const uint8_t* __restrict__ R, int M, int N, const unsigned long long* __restrict__ rmax,
    const unsigned long long* __restrict__ cmax, int pa, int pb, const __grid_constant__ CrtTab tab,
    double* D, int64_t ldd, const double* C, int64_t ldc, double alpha, double beta, double diag,
    int64_t doff, double* __restrict__ sq) {
  double ss = 0.0;  // sum of squares of this thread's stored values (sq != null)
  const int chunks = (N + 3) >> 2;
  const int64_t total = (int64_t)M * chunks;
  const int64_t plane = (int64_t)M * N;
  const bool vec_cd = ((ldd & 1) == 0) && ((reinterpret_cast<uintptr_t>(D) & 15u) == 0) &&
                      (beta == 0.0 || (((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15u) == 0)));
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx / chunks);
    const int j0 = (int)(idx - (int64_t)row * chunks) << 2;
    const int sa = shift_of(rmax[row], pa);
    const int64_t off = (int64_t)row * N + j0;
    const bool full = (j0 + 4 <= N) && ((N & 3) == 0);
    uint32_t w[NMOD];
    if (full) {
#pragma unroll
      for (int l = 0; l < NMOD; ++l) w[l] = __ldcs(reinterpret_cast<const unsigned*>(R + l * plane + off));
    } else {
#pragma unroll
      for (int l = 0; l < NMOD; ++l) {
        w[l] = 0u;
        for (int j = 0; j < 4 && j0 + j < N; ++j) w[l] |= (uint32_t)R[l * plane + off + j] << (8 * j);
      }
    }
    double v[4];
    crt_values4<NMOD>(w, tab, v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = j0 + j;
      const int sb = col < N ? shift_of(cmax[col], pb) : 0;
      v[j] = (sa == kNonFinite || sb == kNonFinite) ? __longlong_as_double(0x7FF8000000000000ll)
                                                    : scale2(v[j], -(sa + sb));
    }
    double* drow = D + (int64_t)row * ldd + j0;
    const double* crow = beta != 0.0 ? C + (int64_t)row * ldc + j0 : nullptr;
    if (full && vec_cd) {
      double cv[4] = {0.0, 0.0, 0.0, 0.0};
      if (crow) {
        const double2 c01 = *reinterpret_cast<const double2*>(crow);
        const double2 c23 = *reinterpret_cast<const double2*>(crow + 2);
        cv[0] = c01.x, cv[1] = c01.y, cv[2] = c23.x, cv[3] = c23.y;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[j] = apply_epi(v[j], alpha, beta, cv[j]);
        if (diag != 0.0 && (int64_t)row + doff == (int64_t)(j0 + j)) v[j] = __dadd_rn(v[j], diag);
      }
      *reinterpret_cast<double2*>(drow) = make_double2(v[0], v[1]);
      *reinterpret_cast<double2*>(drow + 2) = make_double2(v[2], v[3]);
      if (sq) ss = fma(v[3], v[3], fma(v[2], v[2], fma(v[1], v[1], fma(v[0], v[0], ss))));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = j0 + j;
        if (col >= N) break;
        double x = apply_epi(v[j], alpha, beta, crow ? crow[j] : 0.0);
        if (diag != 0.0 && (int64_t)row + doff == (int64_t)col) x = __dadd_rn(x, diag);
        drow[j] = x;
        ss = fma(x, x, ss);
      }
    }
  }
  if (sq) {  // one slot per warp of the (fixed-size) grid: a deterministic partial
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) sq[blockIdx.x * 8 + (threadIdx.x >> 5)] = ss;
  }
}

template <int NMOD>
void launch_crt_n(int blocks, cudaStream_t s, const uint8_t* R, int M, int N,
                  const unsigned long long* rmax, const unsigned long long* cmax, int pa, int pb,
                  const CrtTab& tab, double* D, int64_t ldd, const double* C, int64_t ldc,
                  double alpha, double beta, double diag, int64_t doff, double* sq) {
  crt_kernel<NMOD><<<blocks, 256, 0, s>>>(R, M, N, rmax, cmax, pa, pb, tab, D, ldd, C, ldc, alpha,
                                          beta, diag, doff, sq);
}

template <int NMOD = kMinModuli>
void launch_crt(int nmod, int blocks, cudaStream_t s, const uint8_t* R, int M, int N,
                const unsigned long long* rmax, const unsigned long long* cmax, int pa, int pb,
                const CrtTab& tab, double* D, int64_t ldd, const double* C, int64_t ldc,
                double alpha, double beta, double diag, int64_t doff, double* sq) {
  if constexpr (NMOD <= kMaxModuli) {
    if (nmod == NMOD)
      launch_crt_n<NMOD>(blocks, s, R, M, N, rmax, cmax, pa, pb, tab, D, ldd, C, ldc, alpha, beta,
                         diag, doff, sq);
    else
      launch_crt<NMOD + 1>(nmod, blocks, s, R, M, N, rmax, cmax, pa, pb, tab, D, ldd, C, ldc,
                           alpha, beta, diag, doff, sq);
  }
}

// grid of the CRT kernel for an mc x nc chunk (its sum-of-squares slots: 8 per block)
int crt_blocks(int64_t mc, int64_t nc, int sms) {
  const int64_t thr = mc * ((nc + 3) / 4);
  return (int)std::min<int64_t>((thr + 255) / 256, 64 * sms);
}

// ----------------------------------------------------------------- host --
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// planes x rows x Kp int8, boxes of box_rows x 128 bytes (128B swizzle); rows
// beyond `rows` of a plane read as zeros
bool make_map_i8(CUtensorMap* map, const void* ptr, int64_t Kp, int64_t rows, int planes,
                 uint32_t box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)(rows * Kp)};
  cuuint32_t box[3] = {(cuuint32_t)GBK, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

using u128 = unsigned __int128;

struct Consts {
  ModTab mt;
  CrtTab crt[kMaxModuli + 1];  // by nmod
  int log2m[kMaxModuli + 1];   // floor(log2 M) by nmod
};

const Consts& consts() {
  static Consts c;
  static std::once_flag once;
  std::call_once(once, [] {
    for (int l = 0; l < kMaxModuli; ++l) {
      const unsigned m = kmod(l);
      c.mt.m[l] = m;
      c.mt.magic[l] = (unsigned)((1ull << 39) / m + 1);
      c.mt.off[l] = pow2mod(30, m);
    }
    for (int n = 1; n <= kMaxModuli; ++n) {
      u128 M = 1;
      for (int l = 0; l < n; ++l) M *= kmod(l);
      int bits = 0;
      for (u128 x = M; x > 1; x >>= 1) ++bits;
      c.log2m[n] = bits;  // 2^bits <= M
      CrtTab& t = c.crt[n];
      std::memset(&t, 0, sizeof(t));
      t.nmod = n;
      for (int l = 0; l < n; ++l) {
        const unsigned m = kmod(l);
        const u128 Ml = M / m;
        const unsigned r = (unsigned)(Ml % m);
        unsigned y = 0;
        for (unsigned cand = 1; cand < m; ++cand)
          if ((r * cand) % m == 1u) {
            y = cand;
            break;
          }
        const u128 W = (Ml * y) % M;  // Ml * y < M * 256 / 173 < 2^127
        for (int k = 0; k < 4; ++k) t.w[l][k] = (double)(uint32_t)(W >> (32 * k));
      }
      for (int k = 0; k < 4; ++k) t.mp[k] = (double)(uint32_t)(M >> (32 * k));
      const double md = (double)(uint64_t)(M >> 64) * 0x1p64 + (double)(uint64_t)M;
      t.inv_m = 1.0 / md;
    }
  });
  return c;
}

// rasterisation group and L2 policies of the pair kernel (tuning hook: si_ozaki_tune)
std::atomic<int> g_pair_group_m{8}, g_pair_l2a{0}, g_pair_l2b{0};  // pair: 2048-row groups
std::atomic<int> g_single_group_m{GROUP_M};
std::atomic<int> g_pair_stages{4};  // smem ring depth of the pair kernel (3..6; tuning hook)
std::atomic<int64_t> g_ksplit{0};  // longest K range of one single-CTA launch (0: no split)

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

cudaError_t set_gemm_attr() {
  static std::atomic<uint64_t> done{0};  // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && (done.load() & (1ull << dev))) return cudaSuccess;
  cudaError_t e =
      cudaFuncSetAttribute(i8_gemm_mod_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           GSMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(i8_gemm_mod_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             GSMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(i8_gemm_mod_pair_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             psmem(3));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(i8_gemm_mod_pair_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             psmem(4));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(i8_gemm_mod_pair_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             psmem(5));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(i8_gemm_mod_pair_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             psmem(6));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(i8_gemm_mod_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             GSMEM);
  if (e == cudaSuccess && dev < 64) done.fetch_or(1ull << dev);
  return e;
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
inline int64_t kpad(int64_t K) { return (K + GBK - 1) / GBK * GBK; }

}  // namespace

unsigned modulus(int l) { return kmod(l); }

void tune_ksplit(int64_t kmax) { g_ksplit = kmax > 0 ? kmax : 0; }

void tune_pair_stages(int stages) {
  if (stages >= 3 && stages <= 6) g_pair_stages = stages;
}

void tune_pair(int group_m, int l2a, int l2b) {
  if (group_m > 0) {
    g_pair_group_m = group_m;
    g_single_group_m = group_m;
  }
  if (l2a >= 0 && l2a <= 2) g_pair_l2a = l2a;
  if (l2b >= 0 && l2b <= 2) g_pair_l2b = l2b;
}

namespace {
// columns of D per chunk: B-side planes (nmod x Nc x Kp) + result planes
// (nmod x M x Nc) within kChunkBudget, a multiple of the INT8 tile width
int64_t chunk_cols(int64_t M, int64_t N, int64_t Kp, int nmod, int64_t max_cols) {
  const size_t per_col = (size_t)nmod * (size_t)(Kp + M);
  int64_t fit = std::max<int64_t>(GBN, (int64_t)(kChunkBudget / per_col) / GBN * GBN);
  if (max_cols > 0) fit = std::min(fit, std::max<int64_t>(GBN, max_cols / GBN * GBN));
  if (fit >= N) return N;
  const int64_t nch = (N + fit - 1) / fit;
  const int64_t nc = ((N + nch - 1) / nch + GBN - 1) / GBN * GBN;  // balanced chunks
  return std::min(nc, N);
}
}  // namespace

int64_t chunk_rows(int64_t M, int64_t max_rows) {
  if (max_rows <= 0 || max_rows >= M) return M;
  const int64_t fit = std::max<int64_t>(PBM, max_rows / PBM * PBM);
  const int64_t nch = (M + fit - 1) / fit;
  return std::min(M, ((M + nch - 1) / nch + PBM - 1) / PBM * PBM);  // balanced chunks
}

size_t side_bytes(int64_t rows, int64_t K, int nmod) {
  return align256(rows * 8) + align256((size_t)nmod * rows * kpad(K));
}

size_t workspace_bytes(int64_t M, int64_t N, int64_t K, int nmod, int64_t max_cols,
                       int64_t max_rows) {
  const int64_t Kp = kpad(K);
  const int64_t mc = chunk_rows(M, max_rows);
  const int64_t nc = chunk_cols(mc, N, Kp, nmod, max_cols);
  return align256(mc * 8) + align256(nc * 8) + align256((size_t)nmod * mc * Kp) +
         align256((size_t)nmod * nc * Kp) + align256((size_t)nmod * mc * nc);
}

// kernel launches launch_i8_gemm_mod makes for one call (the K ranges)
static int i8_launch_count(int64_t Kp, int variant) {
  if (variant == kI8Pair || variant == kI8Multicast) return 1;
  const int kblocks = (int)(Kp / GBK);
  const int64_t ks = g_ksplit.load();
  const int maxb = ks > 0 ? (int)std::max<int64_t>(1, ks / GBK) : kblocks;
  const int nranges = (kblocks + maxb - 1) / maxb;
  const int per = (kblocks + nranges - 1) / nranges;
  return (kblocks + per - 1) / per;
}

cudaError_t launch_i8_gemm_mod(const int8_t* A, const int8_t* Bt, uint8_t* R, int64_t M, int64_t N,
                               int64_t Kp, int nplanes, cudaStream_t s, int variant) {
  if (M <= 0 || N <= 0 || Kp <= 0 || Kp % GBK || nplanes < 1 || nplanes > kMaxModuli ||
      M > INT32_MAX || N > INT32_MAX || Kp > kMaxK + GBK || variant < 0 || variant > 3)
    return cudaErrorInvalidValue;
  const bool pair = variant == kI8Pair;  // auto: single CTAs (fewer DRAM bytes; faster at the power cap)
  const bool mc = variant == kI8Multicast;
  CUtensorMap ta, tb;
  if (!make_map_i8(&ta, A, Kp, M, nplanes, pair ? PBM / 2 : GBM) ||
      !make_map_i8(&tb, Bt, Kp, N, nplanes, (pair || mc) ? PBN / 2 : GBN)) {
    set_error("cuTensorMapEncodeTiled failed (int8 planes)");
    return cudaErrorInvalidValue;
  }
  cudaError_t e = set_gemm_attr();
  if (e != cudaSuccess) return e;
  const int sms = num_sms();
  if (pair) {
    const int64_t tiles = ((M + PBM - 1) / PBM) * ((N + PBN - 1) / PBN) * nplanes;
    const int grid = (int)std::min<int64_t>(2 * tiles, sms & ~1);
    const int st = g_pair_stages.load();
    auto kern = st == 3 ? i8_gemm_mod_pair_kernel<3>
                : st == 5 ? i8_gemm_mod_pair_kernel<5>
                : st == 6 ? i8_gemm_mod_pair_kernel<6> : i8_gemm_mod_pair_kernel<4>;
    kern<<<grid, GTHREADS, psmem(st == 3 || st == 5 || st == 6 ? st : 4), s>>>(
        ta, tb, R, (int)M, (int)N, (int)Kp, nplanes, consts().mt, g_pair_group_m.load(),
        g_pair_l2a.load(), g_pair_l2b.load());
  } else if (mc) {
    const int64_t tiles = ((M + 2 * GBM - 1) / (2 * GBM)) * ((N + GBN - 1) / GBN) * nplanes;
    const int grid = (int)std::min<int64_t>(2 * tiles, sms & ~1);
    i8_gemm_mod_mc_kernel<<<grid, GTHREADS, GSMEM, s>>>(ta, tb, R, (int)M, (int)N, (int)Kp,
                                                        nplanes, consts().mt,
                                                        g_single_group_m.load());
  } else {
    const int64_t tiles = ((M + GBM - 1) / GBM) * ((N + GBN - 1) / GBN) * nplanes;
    const int grid = (int)(tiles < sms ? tiles : sms);
    // K split (tuning hook, off by default): K can run as ranges of <= g_ksplit,
    // each later range adding the residues already in R before its reduction
    // -- the same integers mod m_l, bitwise.  Measured at config 5 (K = 32768,
    // where one launch moves 153 GB of DRAM bytes) it did not pay: two ranges
    // of 16384 moved 2 x 118 GB and the step was 1% slower
    // (profiles/ozaki_ksplit_r02.txt).
    const int kblocks = (int)(Kp / GBK);
    const int64_t ks = g_ksplit.load();
    const int maxb = ks > 0 ? (int)std::max<int64_t>(1, ks / GBK) : kblocks;
    const int nranges = (kblocks + maxb - 1) / maxb;
    const int per = (kblocks + nranges - 1) / nranges;  // balanced ranges
    for (int kb0 = 0; kb0 < kblocks; kb0 += per) {
      auto kern = kb0 > 0 ? i8_gemm_mod_kernel<true> : i8_gemm_mod_kernel<false>;
      kern<<<grid, GTHREADS, GSMEM, s>>>(ta, tb, R, (int)M, (int)N, kb0,
                                         std::min(per, kblocks - kb0), nplanes, consts().mt,
                                         g_single_group_m.load());
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_gemm(const Mat& A, const Mat& B, Mat& D, const Epilogue& e, int nmod,
                        const Work& w, cudaStream_t s, int64_t* launches, const I8Hook& hook,
                        Side* a_side, Side* b_side, const RowHook& row_hook) {
  const int64_t M = D.rows, N = D.cols, K = A.cols;
  if (nmod < kMinModuli || nmod > kMaxModuli || K < 1 || K > kMaxK || M > INT32_MAX ||
      N > INT32_MAX || w.bytes < workspace_bytes(M, N, K, nmod, w.max_cols, w.max_rows))
    return cudaErrorInvalidValue;
  const Consts& cs = consts();
  const int64_t Kp = kpad(K);
  const int64_t MC = chunk_rows(M, w.max_rows);
  const int64_t NC = chunk_cols(MC, N, Kp, nmod, w.max_cols);
  int lk = 0;
  while ((1ll << lk) < K) ++lk;
  const int T = cs.log2m[nmod] - 2 - lk;  // K 2^(pa+pb) <= 2^(log2 M - 2) <= M / 4
  const int pa = std::min(kMaxP, (T + 1) / 2), pb = std::min(kMaxP, T / 2);
  uint8_t* p = w.base;
  auto* rmax = reinterpret_cast<unsigned long long*>(p);
  p += align256(MC * 8);
  auto* cmax = reinterpret_cast<unsigned long long*>(p);
  p += align256(NC * 8);
  auto* ares = reinterpret_cast<int8_t*>(p);
  p += align256((size_t)nmod * MC * Kp);
  auto* bres = reinterpret_cast<int8_t*>(p);
  p += align256((size_t)nmod * NC * Kp);
  auto* res = p;
  int64_t n = 0, sq_off = 0;
  cudaError_t err;
  const int sms = num_sms();
  // operand sides kept by the caller (unchunked sides only)
  const bool a_ext = a_side && a_side->scale && a_side->planes && MC == M;
  const bool b_ext = b_side && b_side->scale && b_side->planes && NC == N;
  if (a_ext) {
    rmax = a_side->scale;
    ares = a_side->planes;
  }
  if (b_ext) {
    cmax = b_side->scale;
    bres = b_side->planes;
  }
  for (int64_t i0 = 0; i0 < M; i0 += MC) {
    const int64_t mc = std::min(MC, M - i0);
    const double* ap = A.p + i0 * A.ld;
    if (row_hook) row_hook(i0, i0 + mc);
    // A side of this row chunk: row scales and residue planes
    if (!(a_ext && a_side->ready)) {
      row_absmax_kernel<<<(int)std::min<int64_t>((mc + 7) / 8, 16 * sms), 256, 0, s>>>(
          ap, A.ld, (int)mc, (int)K, rmax);
      ++n;
      const int64_t thr = mc * (Kp / RE);
      const int blocks = (int)std::min<int64_t>((thr + 255) / 256, 64 * sms);
      residues_rows_kernel<<<blocks, 256, 0, s>>>(ap, A.ld, (int)mc, (int)K, (int)Kp, rmax, pa,
                                                   nmod, ares);
      ++n;
      if (a_ext) a_side->ready = true;
    }
    // B side (kept across row chunks when one column chunk covers N), the
    // tensor-core products and the reconstruction per column chunk
    for (int64_t j0 = 0; j0 < N; j0 += NC) {
      const int64_t nc = std::min(NC, N - j0);
      if ((i0 == 0 || NC < N) && !(b_ext && b_side->ready)) {
        const double* bp = B.p + j0;
        if ((err = cudaMemsetAsync(cmax, 0, nc * 8, s)) != cudaSuccess) return err;
        col_absmax_kernel<<<dim3((unsigned)((nc + 31) / 32), (unsigned)((K + 255) / 256)), 256, 0,
                            s>>>(bp, B.ld, (int)K, (int)nc, cmax);
        ++n;
        residues_cols_kernel<<<dim3((unsigned)((nc + 63) / 64), (unsigned)(Kp / 64)), 256, 0, s>>>(
            bp, B.ld, (int)K, (int)nc, (int)Kp, cmax, pb, nmod, bres);
        ++n;
        if (b_ext) b_side->ready = true;
      }
      if ((err = cudaGetLastError()) != cudaSuccess) return err;
      if (hook) hook(true, 2.0 * (double)mc * (double)nc * (double)Kp * (double)nmod);
      if ((err = launch_i8_gemm_mod(ares, bres, res, mc, nc, Kp, nmod, s, w.variant)) !=
          cudaSuccess)
        return err;
      if (hook) hook(false, 0.0);
      n += i8_launch_count(Kp, w.variant);
      const int blocks = crt_blocks(mc, nc, sms);
      launch_crt(nmod, blocks, s, res, (int)mc, (int)nc, rmax, cmax, pa, pb, cs.crt[nmod],
                 D.p + i0 * D.ld + j0, D.ld, e.beta != 0.0 ? e.c + i0 * e.ldc + j0 : nullptr,
                 e.ldc, e.alpha, e.beta, e.diag, e.doff + i0 - j0, e.sq ? e.sq + sq_off : nullptr);
      sq_off += 8 * (int64_t)blocks;
      ++n;
    }
  }
  if (launches) *launches += n;
  return cudaGetLastError();
}

int64_t sq_slots(int64_t M, int64_t N, int64_t K, int nmod, const Work& w) {
  const int64_t MC = chunk_rows(M, w.max_rows);
  const int64_t NC = chunk_cols(MC, N, kpad(K), nmod, w.max_cols);
  const int sms = num_sms();
  int64_t slots = 0;
  for (int64_t i0 = 0; i0 < M; i0 += MC)
    for (int64_t j0 = 0; j0 < N; j0 += NC)
      slots += 8 * (int64_t)crt_blocks(std::min(MC, M - i0), std::min(NC, N - j0), sms);
  return slots;
}

}  // namespace oz
}  // namespace si
