// Batched small systems (BASELINE config 2): thousands of independent n <= 32
// SPD systems, each advanced by `iters` x { plain Richardson update (SURVEY
// a12, ordered as richardson.py:88-89), composite_step (newton_schulz.py:
// 177-228) }.
//
// The per-iteration GEMM DAG is recorded once on the host by the same
// evaluator structure as the dense engine (series_toolkit.py:263-457 over the
// decoded plans), register-allocated onto shared-memory matrix slots, and then
// interpreted by one CTA per system: every matrix stays resident in shared
// memory for all iterations, products run on DMMA (m8n8k4), and HBM is touched
// once per system on entry (coalesced double2 loads) and once on exit.
#include <algorithm>
#include <map>

#include "batched.hpp"

namespace si {
namespace {

constexpr int NPAD = 32;   // systems are zero-padded to 32 x 32
constexpr int LDS = 36;    // shared row stride (doubles): conflict-free fragments
constexpr int MSLOT = NPAD * LDS;
constexpr int BTHREADS = 128;

enum : int8_t { OP_GEMM = 0, OP_GEMV = 1, OP_LIN = 2 };

struct BOp {
  int8_t kind;
  int8_t vec;     // lin over vectors
  int8_t nterms;
  int8_t pad_;
  int16_t dst, a, b, c;
  double alpha, beta, diag;
  int16_t t[kMaxLinTerms];
  double coef[kMaxLinTerms];
};

// ------------------------------------------------------------------ recorder
struct Rec {
  std::vector<BOp> ops;
  std::vector<bool> is_vec;
  int fresh(bool vec) {
    is_vec.push_back(vec);
    return (int)is_vec.size() - 1;
  }
  int gemm(int a, int b, double alpha = 1.0, int c = -1, double beta = 0.0, double diag = 0.0) {
    BOp o{};
    o.kind = OP_GEMM;
    o.a = a;
    o.b = b;
    o.c = c;
    o.alpha = alpha;
    o.beta = c >= 0 ? beta : 0.0;
    o.diag = diag;
    o.dst = fresh(false);
    ops.push_back(o);
    return o.dst;
  }
  int gemv(int a, int v, double alpha, int c, double beta) {
    BOp o{};
    o.kind = OP_GEMV;
    o.a = a;
    o.b = v;
    o.c = c;
    o.alpha = alpha;
    o.beta = c >= 0 ? beta : 0.0;
    o.dst = fresh(true);
    ops.push_back(o);
    return o.dst;
  }
  int lin(double cdiag, const std::vector<std::pair<double, int>>& terms, bool vec) {
    BOp o{};
    o.kind = OP_LIN;
    o.vec = vec;
    o.diag = cdiag;
    o.nterms = (int8_t)terms.size();
    for (size_t i = 0; i < terms.size(); ++i) {
      o.coef[i] = terms[i].first;
      o.t[i] = (int16_t)terms[i].second;
    }
    o.a = o.b = o.c = -1;
    o.dst = fresh(vec);
    ops.push_back(o);
    return o.dst;
  }
  int copy(int x) { return lin(0.0, {{1.0, x}}, is_vec[x]); }
  int residual(int x, int A) { return gemm(x, A, -1.0, -1, 0.0, 1.0); }
  int horner(int y, int x, int h) {
    int z = x;
    for (int i = 0; i < h - 1; ++i) z = gemm(y, z, 1.0, x, 1.0);
    return z;
  }
  int program(const PlanNode& node, int y, int x, int A) {
    std::vector<int> env(node.nregs, -1);
    env[0] = y;
    env[1] = x;
    int res = x;
    for (const Instr& in : node.prog) {
      if (in.op == 0)
        env[in.dst] = gemm(env[in.a], env[in.b]);
      else if (in.op == 1)
        env[in.dst] = residual(env[in.a], A);
      else {
        std::vector<std::pair<double, int>> t;
        for (auto& tt : in.terms) t.emplace_back(tt.first, env[tt.second]);
        env[in.dst] = lin(in.cconst, t, false);
      }
      res = env[in.dst];
    }
    return res;
  }
  int eval(const PlanNode& node, int y, int x, int A) {
    switch (node.kind) {
      case 0:
        return horner(y, x, node.h);
      case 1: {
        int u = node.p == 0 ? x : eval(*node.inner, y, x, A);
        if (node.w == 1) return u;
        int q = node.p == 0 ? y : residual(u, A);
        return eval(*node.outer, q, u, A);
      }
      case 2: {
        int z = eval(*node.inner, y, x, A);
        return gemm(y, z, 1.0, x, 1.0);
      }
      default:
        return program(node, y, x, A);
    }
  }
  int mat_pow(int y, int e) {
    int base = y, result = -1;
    while (e > 0) {
      if (e & 1) result = result < 0 ? base : gemm(result, base);
      e >>= 1;
      if (e) base = gemm(base, base);
    }
    return result;
  }
  int geometric(int y, int x, int order, int A, const PlanNode* base) {
    if (order == 1) return copy(x);
    if (order <= 64) {
      if (!base || plan_order_of(*base) != order) throw Error(kEInval, "missing plan for rate");
      return eval(*base, y, x, A);
    }
    const int half = order / 2;
    int t = geometric(y, x, half, A, base);
    int yh = mat_pow(y, half);
    int z = gemm(yh, t, 1.0, t, 1.0);
    if (order % 2) z = gemm(y, z, 1.0, x, 1.0);
    return z;
  }
};

// Linear-scan assignment of virtual registers to physical slots.
struct Alloc {
  std::vector<int16_t> phys;
  int nmat = 0, nvec = 0;
};

Alloc assign(const Rec& r, const std::vector<int>& pinned, int nops_iter) {
  const int nv = (int)r.is_vec.size();
  std::vector<int> last(nv, -1);
  auto use = [&](int v, int i) {
    if (v >= 0) last[v] = std::max(last[v], i);
  };
  for (int i = 0; i < (int)r.ops.size(); ++i) {
    const BOp& o = r.ops[i];
    use(o.a, i);
    use(o.b, i);
    use(o.c, i);
    if (o.kind == OP_LIN)
      for (int j = 0; j < o.nterms; ++j) use(o.t[j], i);
  }
  for (int p : pinned) last[p] = INT32_MAX;
  (void)nops_iter;
  Alloc al;
  al.phys.assign(nv, -1);
  std::vector<int> free_m, free_v;
  auto take = [&](bool vec) -> int {
    auto& fl = vec ? free_v : free_m;
    if (!fl.empty()) {
      int s = fl.back();
      fl.pop_back();
      return s;
    }
    return vec ? al.nvec++ : al.nmat++;
  };
  for (int p : pinned) al.phys[p] = (int16_t)take(r.is_vec[p]);
  for (int i = 0; i < (int)r.ops.size(); ++i) {
    const BOp& o = r.ops[i];
    al.phys[o.dst] = (int16_t)take(r.is_vec[o.dst]);
    auto release = [&](int v) {
      if (v >= 0 && last[v] == i && al.phys[v] >= 0) {
        (r.is_vec[v] ? free_v : free_m).push_back(al.phys[v]);
        last[v] = -2;  // released once
      }
    };
    release(o.a);
    release(o.b);
    release(o.c);
    if (o.kind == OP_LIN)
      for (int j = 0; j < o.nterms; ++j) release(o.t[j]);
    if (last[o.dst] == -1) {  // never read: free immediately
      (r.is_vec[o.dst] ? free_v : free_m).push_back(al.phys[o.dst]);
    }
  }
  return al;
}

// ------------------------------------------------------------------ device
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double epi(double acc, double alpha, double beta, double cv) {
  double v = (alpha == 1.0) ? acc : (alpha == -1.0 ? -acc : __dmul_rn(alpha, acc));
  if (beta != 0.0) v = __dadd_rn(v, beta == 1.0 ? cv : __dmul_rn(beta, cv));
  return v;
}

struct BatchArgs {
  const double* a;
  const double* b;
  const double* precond;
  const double* residual;
  double* p_io;
  double* f_io;
  double* theta_io;
  const BOp* ops;
  int nops;
  int nmat;
  int n;
  int iters;
  int64_t batch;
  // slots of the pinned registers
  int sA, sP, sB, sG, sF, sT, sb;
  // per-iteration result slots copied back into sG/sF/sT
  int rG, rF, rT;
};

__device__ __forceinline__ double* mslot(double* sm, int s) { return sm + (size_t)s * MSLOT; }
__device__ __forceinline__ double* vslot(double* sm, int nmat, int s) {
  return sm + (size_t)nmat * MSLOT + (size_t)s * NPAD;
}

__device__ void load_mat(double* dst, const double* src, int n) {
  if (n == NPAD) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    for (int i = threadIdx.x; i < NPAD * NPAD / 2; i += BTHREADS) {
      const double2 v = __ldg(s2 + i);
      const int r = (2 * i) / NPAD, c = (2 * i) % NPAD;
      dst[r * LDS + c] = v.x;
      dst[r * LDS + c + 1] = v.y;
    }
  } else {
    for (int i = threadIdx.x; i < NPAD * NPAD; i += BTHREADS) {
      const int r = i / NPAD, c = i % NPAD;
      dst[r * LDS + c] = (r < n && c < n) ? src[r * n + c] : 0.0;
    }
  }
}
__device__ void store_mat(double* dst, const double* src, int n) {
  if (n == NPAD) {
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int i = threadIdx.x; i < NPAD * NPAD / 2; i += BTHREADS) {
      const int r = (2 * i) / NPAD, c = (2 * i) % NPAD;
      d2[i] = make_double2(src[r * LDS + c], src[r * LDS + c + 1]);
    }
  } else {
    for (int i = threadIdx.x; i < n * n; i += BTHREADS) dst[i] = src[(i / n) * LDS + (i % n)];
  }
}

__global__ void __launch_bounds__(BTHREADS) batched_kernel(BatchArgs p) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n = p.n;
  const int64_t nn = (int64_t)n * n;
  for (int64_t sys = blockIdx.x; sys < p.batch; sys += gridDim.x) {
    load_mat(mslot(sm, p.sA), p.a + sys * nn, n);
    load_mat(mslot(sm, p.sP), p.precond + sys * nn, n);
    load_mat(mslot(sm, p.sB), p.residual + sys * nn, n);
    load_mat(mslot(sm, p.sG), p.p_io + sys * nn, n);
    load_mat(mslot(sm, p.sF), p.f_io + sys * nn, n);
    if (threadIdx.x < NPAD) {
      vslot(sm, p.nmat, p.sT)[threadIdx.x] = threadIdx.x < n ? p.theta_io[sys * n + threadIdx.x] : 0.0;
      vslot(sm, p.nmat, p.sb)[threadIdx.x] = threadIdx.x < n ? p.b[sys * n + threadIdx.x] : 0.0;
    }
    __syncthreads();
    for (int it = 0; it < p.iters; ++it) {
      for (int k = 0; k < p.nops; ++k) {
        const BOp& o = p.ops[k];
        if (o.kind == OP_GEMM) {
          const double* A = mslot(sm, o.a);
          const double* B = mslot(sm, o.b);
          const double* C = o.c >= 0 ? mslot(sm, o.c) : nullptr;
          double* D = mslot(sm, o.dst);
          const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 16;
          double acc[2][2][2] = {};
#pragma unroll
          for (int kk = 0; kk < NPAD; kk += 4) {
            double af[2], bf[2];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) af[mi] = A[(r0 + mi * 8 + g) * LDS + kk + t];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) bf[ni] = B[(kk + t) * LDS + c0 + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
          }
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int row = r0 + mi * 8 + g, col = c0 + ni * 8 + 2 * t + h;
                double v = epi(acc[mi][ni][h], o.alpha, o.beta, C ? C[row * LDS + col] : 0.0);
                if (o.diag != 0.0 && row == col && row < n) v = __dadd_rn(v, o.diag);
                D[row * LDS + col] = v;
              }
        } else if (o.kind == OP_GEMV) {
          if (warp == 0) {
            const double* A = mslot(sm, o.a);
            const double* x = vslot(sm, p.nmat, o.b);
            double s = 0.0;
            for (int j = 0; j < NPAD; ++j) {
              const int k2 = (j + lane) & (NPAD - 1);  // rotated: conflict-free
              s = fma(A[lane * LDS + k2], x[k2], s);
            }
            const double cv = o.c >= 0 ? vslot(sm, p.nmat, o.c)[lane] : 0.0;
            vslot(sm, p.nmat, o.dst)[lane] = epi(s, o.alpha, o.beta, cv);
          }
        } else {
          if (o.vec) {
            if (threadIdx.x < NPAD) {
              double acc = 0.0;
              for (int j = 0; j < o.nterms; ++j) {
                const double xv = vslot(sm, p.nmat, o.t[j])[threadIdx.x];
                acc = __dadd_rn(acc, o.coef[j] == 1.0 ? xv : __dmul_rn(o.coef[j], xv));
              }
              vslot(sm, p.nmat, o.dst)[threadIdx.x] = acc;
            }
          } else {
            double* D = mslot(sm, o.dst);
            for (int i = threadIdx.x; i < NPAD * NPAD; i += BTHREADS) {
              const int r = i / NPAD, c = i % NPAD;
              double acc = (r == c && r < n) ? o.diag : 0.0;
              for (int j = 0; j < o.nterms; ++j) {
                const double xv = mslot(sm, o.t[j])[r * LDS + c];
                acc = __dadd_rn(acc, o.coef[j] == 1.0 ? xv : __dmul_rn(o.coef[j], xv));
              }
              D[r * LDS + c] = acc;
            }
          }
        }
        __syncthreads();
      }
      // carry the state: G <- G', F <- F', theta <- theta'
      for (int i = threadIdx.x; i < NPAD * NPAD; i += BTHREADS) {
        const int r = i / NPAD, c = i % NPAD;
        mslot(sm, p.sG)[r * LDS + c] = mslot(sm, p.rG)[r * LDS + c];
        mslot(sm, p.sF)[r * LDS + c] = mslot(sm, p.rF)[r * LDS + c];
      }
      if (threadIdx.x < NPAD) vslot(sm, p.nmat, p.sT)[threadIdx.x] = vslot(sm, p.nmat, p.rT)[threadIdx.x];
      __syncthreads();
    }
    store_mat(p.p_io + sys * nn, mslot(sm, p.sG), n);
    store_mat(p.f_io + sys * nn, mslot(sm, p.sF), n);
    if (threadIdx.x < n) p.theta_io[sys * n + threadIdx.x] = vslot(sm, p.nmat, p.sT)[threadIdx.x];
    __syncthreads();
  }
}

int num_sms_b() {
  static int n = 0;
  if (!n) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  }
  return n;
}

}  // namespace

Counters batched_composite_richardson(Ctx& c, int64_t batch, int64_t n, const double* a,
                                      const double* b, const double* precond,
                                      const double* residual, const std::vector<int>& rates,
                                      const std::vector<const PlanNode*>& plans, int order_n,
                                      int iters, double* p_io, double* f_io, double* theta_io) {
  Rec r;
  const int A = r.fresh(false), P = r.fresh(false), B = r.fresh(false), G = r.fresh(false),
            F = r.fresh(false), T = r.fresh(true), bv = r.fresh(true);
  // plain Richardson with P_k (before the inversion update)
  const int res = r.gemv(A, T, 1.0, bv, -1.0);    // A theta - b
  const int tn = r.gemv(G, res, -1.0, T, 1.0);    // theta - P resid
  // composite_step (ns:177-228)
  std::vector<int> ts, gs;
  for (size_t i = 0; i < rates.size(); ++i) {
    const int ti = r.geometric(B, P, rates[i], A, plans[i]);
    ts.push_back(ti);
    gs.push_back(r.residual(ti, A));
  }
  int tc = ts[0], rc = gs[0];
  for (size_t i = 1; i < ts.size(); ++i) {
    tc = r.gemm(rc, ts[i], 1.0, tc, 1.0);
    rc = r.gemm(rc, gs[i]);
  }
  const int nsp = r.horner(F, G, order_n);
  const int gn = r.gemm(rc, nsp, 1.0, tc, 1.0);
  const int fn = r.residual(gn, A);

  Counters per;
  for (const BOp& o : r.ops) {
    if (o.kind == OP_GEMM) per.mmm += 1;
    if (o.kind == OP_GEMV) per.mvm += 1;
  }
  per.mmm *= iters;
  per.mvm *= iters;
  if (batch == 0 || iters == 0) return per;

  Alloc al = assign(r, {A, P, B, G, F, T, bv, gn, fn, tn}, (int)r.ops.size());
  std::vector<BOp> ops = r.ops;
  auto ph = [&](int v) -> int16_t { return v >= 0 ? al.phys[v] : (int16_t)-1; };
  for (BOp& o : ops) {
    o.dst = ph(o.dst);
    o.a = ph(o.a);
    o.b = ph(o.b);
    o.c = ph(o.c);
    if (o.kind == OP_LIN)
      for (int j = 0; j < o.nterms; ++j) o.t[j] = ph(o.t[j]);
  }
  const size_t smem = (size_t)al.nmat * MSLOT * sizeof(double) + (size_t)al.nvec * NPAD * sizeof(double);
  if (smem > 227 * 1024) throw Error(kEInval, "batched program needs too much shared memory");

  MV dops = alloc(c, (int64_t)((ops.size() * sizeof(BOp) + 7) / 8), 1);
  check(cudaMemcpyAsync(dops.v.p, ops.data(), ops.size() * sizeof(BOp), cudaMemcpyHostToDevice, c.s),
        "memcpy program");
  BatchArgs args;
  args.a = a;
  args.b = b;
  args.precond = precond;
  args.residual = residual;
  args.p_io = p_io;
  args.f_io = f_io;
  args.theta_io = theta_io;
  args.ops = reinterpret_cast<const BOp*>(dops.v.p);
  args.nops = (int)ops.size();
  args.nmat = al.nmat;
  args.n = (int)n;
  args.iters = iters;
  args.batch = batch;
  args.sA = al.phys[A];
  args.sP = al.phys[P];
  args.sB = al.phys[B];
  args.sG = al.phys[G];
  args.sF = al.phys[F];
  args.sT = al.phys[T];
  args.sb = al.phys[bv];
  args.rG = al.phys[gn];
  args.rF = al.phys[fn];
  args.rT = al.phys[tn];
  check(cudaFuncSetAttribute(batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
        "cudaFuncSetAttribute");
  int per_sm = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batched_kernel, BTHREADS, smem),
        "occupancy");
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = std::min<int64_t>(batch, (int64_t)num_sms_b() * per_sm);
  batched_kernel<<<(unsigned)grid, BTHREADS, smem, c.s>>>(args);
  check(cudaGetLastError(), "batched kernel launch");
  return per;
}

}  // namespace si
