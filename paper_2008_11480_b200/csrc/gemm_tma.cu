// FP64 GEMM for sm_100a: TMA-staged, mbarrier-pipelined, warp-specialised,
// persistent, on the FP64 DMMA tensor path (mma.sync m8n8k4 -> SASS DMMA.8x8x4),
// with the seriesinv epilogue D = alpha*(A@B) + beta*C + diag*I fused.
//
// This is the kernel behind every n x n product of the hot path
// (matrix_core.py:101-106 mat_mul, and the element-wise op that follows each
// product at its call site: series_toolkit.py:265-266, :273, :375-378;
// newton_schulz.py:144,166,210,215-220,268-270,287-288; richardson.py:148-154,168).
//
// Design (B200, 148 SMs, DMMA peak measured at 37.0 TFLOP/s = 64 FMA/clk/SM):
//  * CTA tile 128x128, BK=16 doubles per stage, 6-stage ring (32 KB/stage).
//  * 1 producer warp: one lane issues cp.async.bulk.tensor (TMA) for the A box
//    (16 x 128, 128B swizzle) and up to 8 B boxes (16 x 16, 128B swizzle).
//  * 8 consumer warps (2 x 4), warp tile 64 x 32 = 8 x 4 DMMA tiles, 128 FP64
//    accumulator registers per thread.
//  * Bank-conflict-free fragment loads: the 4 k-lanes of each DMMA read the k
//    rows {0,3,12,15} / {8,11,4,7} / {1,2,13,14} / {9,10,5,6} of the swizzled
//    slab, so every 256 B warp load is exactly 2 shared-memory wavefronts for
//    both operands (see kperm).  The permutation is
//    fixed, so the K accumulation order is deterministic (serial == concurrent
//    bitwise, newton_schulz.py:259-261).
//  * Persistent grid (<= #SMs CTAs), grouped tile rasterisation for L2 reuse;
//    the producer runs ahead into the next tile while consumers drain the
//    epilogue.
//  * Optional row-panel gates on A (per tile rows) and B (per k-slab); used for
//    inputs whose host->device copy is still in flight.
//  * Wave lockstep (multi-wave products): the producer lanes of all CTAs
//    advance through k in epochs of kSyncEpoch k-blocks and a lane may start
//    epoch E only when every CTA has issued epoch E-2 (per-epoch arrival
//    counters in a 4-slot ring).  The CTAs of a wave then read each k-slab of
//    their shared A / B panels within ~2 epochs of each other, so the slab is
//    still in L2 for all of them: without it the CTAs drift apart over a long
//    launch and every CTA streams its panels from HBM (n=32768: 3.2 TB of DRAM
//    traffic per product against a 0.4 TB lockstep floor).  The order in which
//    a tile accumulates k is unchanged, so results are bitwise unchanged; the
//    slowest CTA never waits, and a wait that exceeds 1 ms (CTAs of this grid
//    not yet resident, e.g. beside a concurrent product) turns the throttle off
//    for that CTA rather than stall it.
//  * Optional panel gate (sharded path): when B is a matrix whose row panels
//    are still arriving from peer GPUs (copy engines, flags written by stream
//    memory operations), the producer lane acquires panel p's flag before its
//    first TMA load from that panel -- the gather overlaps the product k-slab
//    by k-slab instead of completing before the launch.
#include "common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <mutex>

namespace si {
namespace {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int STAGES = 6;
constexpr int NUM_CONSUMER_WARPS = 8;  // two consumer warpgroups
// + one producer warpgroup (only one lane issues TMA).  Register budget is
// moved with setmaxnreg: producers drop to 40, consumers rise to 232, which the
// 128 FP64 accumulators plus two buffered fragment sets need.
constexpr int THREADS = (NUM_CONSUMER_WARPS + 4) * 32;
constexpr int PRODUCER_REGS = 40;
constexpr int CONSUMER_REGS = 232;
constexpr int A_STAGE_BYTES = BM * BK * 8;  // 16 KB
constexpr int B_BOX_BYTES = 16 * BK * 8;    // 2 KB (16 cols x 16 rows)
constexpr int B_STAGE_BYTES = BK * BN * 8;  // 16 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8;
constexpr int GROUP_M = 12;  // a wave of 148 tiles: 12 x 12.3 panels (DRAM -8% vs 8 x 18.5)
constexpr int kSyncEpoch = 8;     // k-blocks per lockstep epoch
constexpr int kSyncRing = 4;      // arrival counters per launch (epochs e, e+4, ... share one)
constexpr int kSyncSets = 64;     // counter sets per device, handed out round robin
constexpr int kSyncMinKBlocks = 64;

// One launch's lockstep counters (self-cleaning: the last CTA to finish zeroes them).
struct alignas(64) SyncSet {
  unsigned ring[kSyncRing];
  unsigned done;
  unsigned pad[11];
};

struct WaveSync {
  SyncSet* set = nullptr;  // null: no lockstep (single wave / short K)
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
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Blocks until every row panel overlapping rows [k0, k1) of B has arrived.
// `known` caches the panels already seen.  A flag that has not arrived after
// 60 s means a broken exchange: trap (the launch fails) rather than hang.
__device__ __forceinline__ void panel_gate(const PanelWait& pw, int k0, int k1, uint32_t& known) {
  for (int p = 0; p < pw.npanels; ++p) {
    if (pw.bounds[p + 1] <= k0 || pw.bounds[p] >= k1 || (known >> p) & 1u) continue;
    const uint64_t t0 = globaltimer_ns();
    while ((int)(ld_acquire_u32(pw.ready + p) - pw.epoch) < 0) {
      __nanosleep(256);
      if (globaltimer_ns() - t0 > 60ull * 1000000000ull) __trap();
    }
    known |= 1u << p;
    // the panel was written by a copy engine (generic proxy); TMA reads it
    // through the async proxy
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Arrivals expected in ring slot (e % kSyncRing) once every CTA has issued
// epochs 0..e: CTAs own `hi` = T-tile or `lo` = (T-1)-tile schedules with EH /
// EL epochs each; slot j collects epochs j, j + R, j + 2R, ...
__device__ __forceinline__ unsigned sync_expected(int e, int n_hi, int eh, int n_lo, int el) {
  const int j = e % kSyncRing;
  auto cnt = [&](int epochs) {
    const int m = min(e, epochs - 1);
    return m >= j ? (m - j) / kSyncRing + 1 : 0;
  };
  return (unsigned)(n_hi * cnt(eh) + n_lo * cnt(el));
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// k index supplied by k-lane t (0..3) of k-step s (0..3) inside a 16-deep slab.
// Shared memory serves an 8-byte warp load in two half-warp phases of 128 B;
// with the 128B TMA swizzle (16-B chunk ^= row & 7) a phase is conflict-free
// iff its 16 (chunk, 8-byte half) slots are distinct.  For the A fragment
// (rows g, k = K[t]) that needs K>>1 to differ by 4 between the two k-lanes
// that share K&1; for the B fragment (rows K[t], columns g) it needs (K&7)>>1
// distinct over the four k-lanes.  These four k-sets satisfy both, so every
// fragment load costs the minimum 2 wavefronts.
__device__ __forceinline__ int kperm(int s, int t) {
  // = {0,3,12,15, 8,11,4,7, 1,2,13,14, 9,10,5,6}[4 s + t], computed (no local array)
  return 8 * ((t >> 1) ^ (s & 1)) + (t >> 1) * 4 + ((s >> 1) ? 1 + (t & 1) : 3 * (t & 1));
}

__device__ __forceinline__ double apply_epi(double acc, double alpha, double beta, double cval) {
  double v = (alpha == 1.0) ? acc : (alpha == -1.0 ? -acc : __dmul_rn(alpha, acc));
  if (beta != 0.0) v = __dadd_rn(v, beta == 1.0 ? cval : __dmul_rn(beta, cval));
  return v;
}

__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int group_m, int& tm,
                                            int& tn) {
  const int per_group = group_m * num_n;
  const int group = tile / per_group;
  const int first_m = group * group_m;
  const int gsize = min(num_m - first_m, group_m);
  const int r = tile % per_group;
  tm = first_m + r % gsize;
  tn = r / gsize;
}

template <int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_f64_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, double* __restrict__ D,
                        int64_t ldd, const double* __restrict__ C, int64_t ldc, int M, int N,
                        int K, double alpha, double beta, double diag, int64_t doff,
                        const __grid_constant__ PanelWait pw,
                        const __grid_constant__ PanelWait pwa, SyncSet* __restrict__ sync,
                        int group_m, double* __restrict__ sq) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + STAGES * STAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int kblocks = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), NUM_CONSUMER_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= NUM_CONSUMER_WARPS) {
    // ---------------- TMA producer ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PRODUCER_REGS));
    if (warp == NUM_CONSUMER_WARPS && lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      uint32_t known = pw.ready ? 0u : ~0u;
      uint32_t known_a = pwa.ready ? 0u : ~0u;  // row panels of A (inputs in flight)
      // wave lockstep: this CTA's k-blocks are numbered g = 0, 1, ... across its
      // tiles; epoch g / kSyncEpoch.  Tile counts per CTA are T or T-1.
      bool lockstep = sync != nullptr;
      const int T = (num_tiles + (int)gridDim.x - 1) / (int)gridDim.x;
      const int n_hi = num_tiles - (T - 1) * (int)gridDim.x;
      const int n_lo = (int)gridDim.x - n_hi;
      const int eh = (T * kblocks + kSyncEpoch - 1) / kSyncEpoch;
      const int el = ((T - 1) * kblocks + kSyncEpoch - 1) / kSyncEpoch;
      int g = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int tm, tn;
        tile_coords(tile, num_m, num_n, group_m, tm, tn);
        const int n0 = tn * BN;
        if (~known_a) panel_gate(pwa, tm * BM, min(M, tm * BM + BM), known_a);
        const int nboxes = min(8, (N - n0 + 15) / 16);
        const uint32_t bytes = A_STAGE_BYTES + nboxes * B_BOX_BYTES;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          if (sync != nullptr && g > 0 && g % kSyncEpoch == 0) {
            const int e = g / kSyncEpoch;  // about to start epoch e: epoch e-1 is issued
            atomicAdd(&sync->ring[(e - 1) % kSyncRing], 1u);
            if (lockstep && e >= 2) {
              const unsigned want = sync_expected(e - 2, n_hi, eh, n_lo, el);
              const unsigned* slot = &sync->ring[(e - 2) % kSyncRing];
              if ((int)(ld_relaxed_u32(slot) - want) < 0) {
                const uint64_t t0 = globaltimer_ns();
                while ((int)(ld_relaxed_u32(slot) - want) < 0) {
                  __nanosleep(64);
                  if (globaltimer_ns() - t0 > 1000000ull) {  // 1 ms: stop throttling
                    lockstep = false;
                    break;
                  }
                }
              }
            }
          }
          if (~known) panel_gate(pw, kb * BK, min(K, kb * BK + BK), known);
          mbar_wait(empty_bar(stage), phase ^ 1u);
          const uint32_t sa = base + stage * STAGE_BYTES;
          const uint32_t sb = sa + A_STAGE_BYTES;
          mbar_expect_tx(full_bar(stage), bytes);
          tma_load_2d(sa, &tmA, full_bar(stage), kb * BK, tm * BM);
          for (int j = 0; j < nboxes; ++j)
            tma_load_2d(sb + j * B_BOX_BYTES, &tmB, full_bar(stage), n0 + j * 16, kb * BK);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (EPI == 1 && C != nullptr && beta != 0.0) {
          // the consumers reach this tile's epilogue ~STAGES k-blocks from now:
          // pull its C rows into L2 so the epilogue loads do not wait on HBM
          const int m0 = tm * BM, rows = min(BM, M - m0);
          const uint32_t bytes_row = (uint32_t)(min(BN, N - n0) * 8) & ~15u;
          if (bytes_row)
            for (int r = 0; r < rows; ++r)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                               C + (int64_t)(m0 + r) * ldc + n0),
                           "r"(bytes_row)
                           : "memory");
        }
      }
      if (sync != nullptr) {
        if (g > 0) atomicAdd(&sync->ring[((g - 1) / kSyncEpoch) % kSyncRing], 1u);
        // every arrival and every wait of this CTA is behind this point: the
        // last CTA out leaves the set zeroed for the next launch that draws it
        __threadfence();
        if (atomicAdd(&sync->done, 1u) == gridDim.x - 1) {
          for (int j = 0; j < kSyncRing; ++j) atomicExch(&sync->ring[j], 0u);
          atomicExch(&sync->done, 0u);
        }
      }
    }
    return;
  }

  // ---------------- DMMA consumers ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CONSUMER_REGS));
  const int wm = warp >> 2;  // 0..1 -> 64-row half
  const int wn = warp & 3;   // 0..3 -> 32-col quarter
  const int g = lane >> 2;   // fragment row / col group
  const int t = lane & 3;    // k-lane

  uint32_t a_off[4], b_off[4][2];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int k = kperm(s, t);
    a_off[s] = (wm * 64 + g) * 128 + ((((k >> 1) ^ g) & 7) << 4) + ((k & 1) << 3);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int nl = h * 8 + g;  // column inside a 16-wide box
      b_off[s][h] = wn * 2 * B_BOX_BYTES + k * 128 + ((((nl >> 1) ^ (k & 7)) & 7) << 4) +
                    ((nl & 1) << 3);
    }
  }

  int stage = 0;
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
    int tm, tn;
    tile_coords(tile, num_m, num_n, group_m, tm, tn);
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // Fragments are double-buffered one k-step ahead: the loads of step s+1
    // (and of the next slab's step 0) are in flight while the 32 DMMAs of step s
    // issue, so no DMMA waits on shared-memory latency.
    double fa[2][8], fb[2][4];
    auto load_frags = [&](int buf, uint32_t sa, uint32_t sb, int s) {
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) fa[buf][mi] = lds(sa + a_off[s] + mi * 1024);
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
        fb[buf][ni] = lds(sb + b_off[s][ni & 1] + (ni >> 1) * B_BOX_BYTES);
    };
    auto mma_step = [&](int buf) {
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
          dmma(acc[mi][ni][0], acc[mi][ni][1], fa[buf][mi], fb[buf][ni]);
    };
    mbar_wait(full_bar(stage), phase);
    uint32_t sa = base + stage * STAGE_BYTES;
    uint32_t sb = sa + A_STAGE_BYTES;
    load_frags(0, sa, sb, 0);
    for (int kb = 0; kb < kblocks; ++kb) {
      load_frags(1, sa, sb, 1);
      mma_step(0);
      load_frags(0, sa, sb, 2);
      mma_step(1);
      load_frags(1, sa, sb, 3);
      mma_step(0);
      // every load of this slab has been issued: hand the stage back to TMA
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_bar(stage));
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
      if (kb + 1 < kblocks) {
        mbar_wait(full_bar(stage), phase);
        sa = base + stage * STAGE_BYTES;
        sb = sa + A_STAGE_BYTES;
        load_frags(0, sa, sb, 0);
      }
      mma_step(1);
    }

    // ---------------- fused epilogue ----------------
    const int row0 = tm * BM + wm * 64 + g;
    const int col0 = tn * BN + wn * 32 + 2 * t;
    // sum of squares of the stored values (sq != null): one slot per (tile,
    // consumer warp), written by that warp alone -- a fixed-order reduction
    // of the slots later gives ||D||_F^2 deterministically
    double ss = 0.0;
    auto flush_sq = [&]() {
      if (sq == nullptr) return;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) sq[(int64_t)tile * NUM_CONSUMER_WARPS + warp] = ss;
    };
    if (EPI == 1 && beta != 0.0) {
      // C loads issued a pair of fragment rows ahead of the stores that use them
      // (each thread reads its own elements before writing them, so D == C is fine)
      auto load_c = [&](double2 (&cv)[2][4], int mi0) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = row0 + (mi0 + h) * 8;
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            const int col = col0 + ni * 8;
            cv[h][ni] = make_double2(0.0, 0.0);
            if (row < M && col < N) {
              const double* pc = C + (int64_t)row * ldc + col;
              if (col + 1 < N) cv[h][ni] = *reinterpret_cast<const double2*>(pc);
              else cv[h][ni].x = *pc;
            }
          }
        }
      };
      double2 cbuf[2][2][4];
      load_c(cbuf[0], 0);
#pragma unroll
      for (int mp = 0; mp < 4; ++mp) {
        if (mp + 1 < 4) load_c(cbuf[(mp + 1) & 1], 2 * (mp + 1));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int mi = 2 * mp + h;
          const int row = row0 + mi * 8;
          if (row >= M) continue;
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            const int col = col0 + ni * 8;
            if (col >= N) continue;
            const double2 cv = cbuf[mp & 1][h][ni];
            double v0 = apply_epi(acc[mi][ni][0], alpha, beta, cv.x);
            double v1 = apply_epi(acc[mi][ni][1], alpha, beta, cv.y);
            if (diag != 0.0) {
              if (row + doff == col) v0 = __dadd_rn(v0, diag);
              if (row + doff == col + 1) v1 = __dadd_rn(v1, diag);
            }
            if (col + 1 < N) {
              *reinterpret_cast<double2*>(D + (int64_t)row * ldd + col) = make_double2(v0, v1);
              ss = fma(v1, v1, fma(v0, v0, ss));
            } else {
              D[(int64_t)row * ldd + col] = v0;
              ss = fma(v0, v0, ss);
            }
          }
        }
      }
      flush_sq();
      continue;
    }
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int row = row0 + mi * 8;
      if (row >= M) continue;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int col = col0 + ni * 8;
        if (col >= N) continue;
        double c0 = 0.0, c1 = 0.0;
        const bool two = (col + 1 < N);
        if (beta != 0.0) {
          if (two) {
            const double2 cv = *reinterpret_cast<const double2*>(C + (int64_t)row * ldc + col);
            c0 = cv.x;
            c1 = cv.y;
          } else {
            c0 = C[(int64_t)row * ldc + col];
          }
        }
        double v0 = apply_epi(acc[mi][ni][0], alpha, beta, c0);
        double v1 = apply_epi(acc[mi][ni][1], alpha, beta, c1);
        if (diag != 0.0) {
          if (row + doff == col) v0 = __dadd_rn(v0, diag);
          if (row + doff == col + 1) v1 = __dadd_rn(v1, diag);
        }
        if (two) {
          *reinterpret_cast<double2*>(D + (int64_t)row * ldd + col) = make_double2(v0, v1);
          ss = fma(v1, v1, fma(v0, v0, ss));
        } else {
          D[(int64_t)row * ldd + col] = v0;
          ss = fma(v0, v0, ss);
        }
      }
    }
    flush_sq();
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

bool make_map(CUtensorMap* map, const double* ptr, int64_t rows, int64_t cols, int64_t ld,
              uint32_t box_cols, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// kSyncSets lockstep counter sets per device (zeroed once; every launch
// leaves its set zeroed).  A set is in use for one launch; handing them out
// round robin keeps concurrently running products on different sets.
SyncSet* draw_sync_set(int dev) {
  static std::mutex mu;
  static SyncSet* sets[64] = {};
  static std::atomic<unsigned> next{0};
  if (dev < 0 || dev >= 64) return nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!sets[dev]) {
      void* p = nullptr;
      if (cudaMalloc(&p, kSyncSets * sizeof(SyncSet)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      if (cudaMemset(p, 0, kSyncSets * sizeof(SyncSet)) != cudaSuccess ||
          cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p);
        return nullptr;
      }
      sets[dev] = static_cast<SyncSet*>(p);
    }
  }
  return sets[dev] + next.fetch_add(1) % kSyncSets;
}

// SI_GEMM_LOCKSTEP=0 turns the wave lockstep off (A/B measurements; read once)
bool lockstep_disabled() {
  static const bool off = [] {
    const char* v = std::getenv("SI_GEMM_LOCKSTEP");
    return v != nullptr && v[0] == '0';
  }();
  return off;
}

// Row tiles per rasterisation group (a wave of 148 tiles spans GROUP_M row
// panels x 148 / GROUP_M column panels); SI_GEMM_GROUP_M overrides (A/B
// measurements of DRAM traffic; the tile -> CTA map changes, no result does)
int group_m() {
  static const int g = [] {
    const char* v = std::getenv("SI_GEMM_GROUP_M");
    const int x = v ? std::atoi(v) : GROUP_M;
    return x >= 1 ? x : GROUP_M;
  }();
  return g;
}

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);  // cached by the runtime
  return n;
}

}  // namespace

bool tma_eligible(const Mat& A, const Mat& B, const Mat& D, const Epilogue& e) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (!al16(A.p) || !al16(B.p) || !al16(D.p)) return false;
  if ((A.ld & 1) || (B.ld & 1) || (D.ld & 1)) return false;
  if (e.beta != 0.0 && (!al16(e.c) || (e.ldc & 1))) return false;
  if (A.rows > INT32_MAX || A.cols > INT32_MAX || B.cols > INT32_MAX) return false;
  return get_encode() != nullptr;
}

cudaError_t launch_gemm_tma(const Mat& A, const Mat& B, Mat& D, const Epilogue& e,
                            cudaStream_t s, const PanelWait* pw, const PanelWait* pwa) {
  CUtensorMap ta, tb;
  if (!make_map(&ta, A.p, A.rows, A.cols, A.ld, BK, BM) ||
      !make_map(&tb, B.p, B.rows, B.cols, B.ld, 16, BK)) {
    set_error("cuTensorMapEncodeTiled failed");
    return cudaErrorInvalidValue;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<uint64_t> attr_set{0};  // one bit per device
  if (dev < 64 && !(attr_set.load() & (1ull << dev))) {
    for (auto fn : {gemm_f64_tma_kernel<0>, gemm_f64_tma_kernel<1>}) {
      cudaError_t err =
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      if (err != cudaSuccess) return err;
    }
    attr_set.fetch_or(1ull << dev);
  } else if (dev >= 64) {
    for (auto fn : {gemm_f64_tma_kernel<0>, gemm_f64_tma_kernel<1>}) {
      cudaError_t err =
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      if (err != cudaSuccess) return err;
    }
  }
  const int M = (int)D.rows, N = (int)D.cols, K = (int)A.cols;
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  // lockstep only pays for products of several waves with a long K loop
  const int kblocks = (K + BK - 1) / BK;
  SyncSet* sync = (tiles > grid && kblocks >= kSyncMinKBlocks && !lockstep_disabled())
                      ? draw_sync_set(dev) : nullptr;
  PanelWait gate, gate_a;
  if (pw && pw->ready && pw->npanels > 0) gate = *pw;
  if (pwa && pwa->ready && pwa->npanels > 0) gate_a = *pwa;
  static const int epi = [] {
    const char* v = std::getenv("SI_GEMM_EPI");
    return v ? std::atoi(v) : 1;
  }();
  auto kern = epi == 1 ? gemm_f64_tma_kernel<1> : gemm_f64_tma_kernel<0>;
  kern<<<grid, THREADS, SMEM_BYTES, s>>>(ta, tb, D.p, D.ld, e.c, e.ldc, M, N, K,
                                                        e.alpha, e.beta, e.diag, e.doff, gate,
                                                        gate_a, sync, group_m(), e.sq);
  return cudaGetLastError();
}

int64_t gemm_tma_sq_slots(int64_t M, int64_t N) {
  return ((M + BM - 1) / BM) * ((N + BN - 1) / BN) * NUM_CONSUMER_WARPS;
}

}  // namespace si
