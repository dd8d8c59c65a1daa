// Resident small systems: BASELINE config 2 (16384 independent 32 x 32
// systems, composite step + plain Richardson) and config 1 (one 64 x 64
// system, Newton-Schulz step + plain Richardson).
//
// One iteration of the reference GEMM DAG (series_toolkit.py:263-457 over the
// decoded plans, newton_schulz.py:150-228, plain Richardson as
// richardson.py:88-89) is recorded once on the host, register-allocated onto
// shared-memory matrix slots, and interpreted by one CTA per system for all
// `iters` iterations: the state never leaves shared memory, products run on
// DMMA (m8n8k4), and HBM is touched once per system on entry and exit (plus
// the splitting S^-1 / B, streamed in when a product needs them so they do
// not occupy slots).  Per system this executes exactly the reference's
// products, so MulCounter deltas match tick for tick.
//
// Shared-memory layout: a slot is an unpadded NP x NP row-major matrix whose
// 16-byte chunks are XOR-swizzled by {0,4,2,6}[row & 3]; every DMMA fragment
// load is then the minimum 2 wavefronts and every accumulator store / C load
// (16 bytes per lane, rows g and g+1 in one quarter-warp) the minimum 4.
// Slots are 8 KB (NP=32) / 32 KB (NP=64); the ops are reordered to minimise
// live slots (32 x 32 products may overwrite their own operands: config 2
// needs 5 slots, 42 KB per CTA); systems are claimed dynamically by the CTAs.
#include <algorithm>
#include <bitset>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <utility>

#include "batched.hpp"

namespace si {
namespace {

enum : int8_t { OP_GEMM = 0, OP_GEMV = 1, OP_LIN = 2, OP_LOAD = 3 };

struct BOp {
  int8_t kind;
  int8_t vec;  // lin over vectors; for OP_LOAD: 0 = S^-1, 1 = B
  int8_t nterms;
  int8_t pad_;
  int16_t dst, a, b, c;
  double alpha, beta, diag;
  int16_t t[kMaxLinTerms];
  double coef[kMaxLinTerms];
};
constexpr int kMaxOps = 96;

// Device form of an op: 32 bytes, read with two 16-byte shared loads.  The
// epilogue variant is decided on the host (`mode`) and the few non-unit
// constants live in a side table (`cidx`), so an op costs no FP64 compares.
//   GEMM mode: 0 A@B, 1 I - A@B, 2 A@B + C, 3 generic (cst: alpha, beta, diag)
//   GEMV mode: 1 A@x - c, 2 c - A@x, 3 generic (cst: alpha, beta)
//   LIN:       cst: cdiag, coef[0..nterms)        LOAD mode: 0 S^-1, 1 B
struct __align__(16) DOp {
  uint8_t kind, mode, sync, nterms;
  int16_t dst, a, b, c;
  int16_t t[kMaxLinTerms];
  int16_t cidx;
  int16_t prebar;  // GEMM writing over its A or B operand: barrier before the stores
  int16_t pad[2];
};
static_assert(sizeof(DOp) == 32, "DOp layout");

// ------------------------------------------------------------------ recorder
struct Rec {
  std::vector<BOp> ops;
  std::vector<bool> is_vec;
  int fresh(bool vec) {
    is_vec.push_back(vec);
    return (int)is_vec.size() - 1;
  }
  int load(int which) {
    BOp o{};
    o.kind = OP_LOAD;
    o.vec = (int8_t)which;
    o.a = o.b = o.c = -1;
    o.dst = fresh(false);
    ops.push_back(o);
    return o.dst;
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
    const auto& prog = node.prog;
    for (size_t i = 0; i < prog.size(); ++i) {
      const Instr& in = prog[i];
      if (in.op == 0 && i + 1 < prog.size()) {
        // Mul followed by "0*I + 1*other + 1*mul" with the product used nowhere
        // else: one GEMM with the add in its epilogue (same rounding).
        const Instr& nx = prog[i + 1];
        bool dead_after = true;
        for (size_t j = i + 2; j < prog.size(); ++j) {
          const Instr& u = prog[j];
          if (u.a == in.dst || u.b == in.dst) dead_after = false;
          for (auto& tt : u.terms)
            if (tt.second == in.dst) dead_after = false;
        }
        if (nx.op == 2 && nx.cconst == 0.0 && nx.terms.size() == 2 && nx.terms[0].first == 1.0 &&
            nx.terms[1].first == 1.0 && dead_after && nx.dst != in.dst &&
            (nx.terms[0].second == in.dst) != (nx.terms[1].second == in.dst)) {
          const int other = nx.terms[0].second == in.dst ? nx.terms[1].second : nx.terms[0].second;
          env[nx.dst] = gemm(env[in.a], env[in.b], 1.0, env[other], 1.0);
          res = env[nx.dst];
          ++i;
          continue;
        }
      }
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

// Operands an op may overwrite in place (dst in the same slot): each element
// is read and then written by the same thread -- the C operand of a product
// (read into the accumulator or in the epilogue), the c vector of a GEMV, the
// terms of a LIN -- and only when it is not also read as A / B / x.  With
// `ab` (the one-CTA-per-system kernel, whose slots no other CTA reads) a
// product may also overwrite its A or B operand: every warp has finished its
// main loop -- the last read of A and B -- at a CTA barrier before the first
// store (DOp::prebar); the C operand is preferred (no barrier).
std::vector<int> inplace_operands(const BOp& o, bool ab = false) {
  std::vector<int> v;
  if (o.kind == OP_GEMM || o.kind == OP_GEMV) {
    if (o.c >= 0 && o.c != o.a && o.c != o.b) v.push_back(o.c);
    if (ab && o.kind == OP_GEMM) {
      if (o.a >= 0 && o.a != o.c) v.push_back(o.a);
      if (o.b >= 0 && o.b != o.c && o.b != o.a) v.push_back(o.b);
    }
  } else if (o.kind == OP_LIN) {
    for (int j = 0; j < o.nterms; ++j) v.push_back(o.t[j]);
  }
  return v;
}

// Reorders the recorded ops (a topological order of the SSA DAG) so that the
// peak number of live matrices -- the shared-memory footprint, hence CTAs per
// SM -- is minimal.  Branch and bound over schedules, ready ops tried in
// recorded order (so the recorded order is the first candidate and is kept on
// ties), memoised on the set of scheduled ops, with a node budget.  Products
// are unchanged, only their order, so every value is bitwise the same.
void schedule_min_live(Rec& r, const std::vector<int>& pinned,
                       const std::vector<std::pair<int, int>>& carried, bool ab) {
  const int nops = (int)r.ops.size(), nv = (int)r.is_vec.size();
  if (nops > 128) return;
  using Mask = std::bitset<128>;
  std::vector<int> producer(nv, -1);
  std::vector<std::vector<int>> reads(nops);  // unique matrix operands
  std::vector<std::vector<int>> deps(nops);
  for (int i = 0; i < nops; ++i) {
    const BOp& o = r.ops[i];
    producer[o.dst] = i;
    std::vector<int> all = {o.a, o.b, o.c};
    if (o.kind == OP_LIN)
      for (int j = 0; j < o.nterms; ++j) all.push_back(o.t[j]);
    for (int v : all) {
      if (v < 0) continue;
      if (!r.is_vec[v] && std::find(reads[i].begin(), reads[i].end(), v) == reads[i].end())
        reads[i].push_back(v);
    }
    for (int v : all)
      if (v >= 0 && producer[v] >= 0 && producer[v] != i) deps[i].push_back(producer[v]);
  }
  std::vector<char> keep(nv, 0);  // never released: pinned values and carried outputs
  for (int v : pinned) keep[v] = 1;
  for (auto& pr : carried) keep[pr.second] = 1;
  std::vector<int> uses(nv, 0);
  for (int i = 0; i < nops; ++i)
    for (int v : reads[i]) uses[v] += 1;
  int live0 = 0;
  for (int v : pinned) live0 += !r.is_vec[v];
  for (auto& pr : carried) live0 += (!r.is_vec[pr.first] && uses[pr.first] > 0);

  std::vector<int> order, best_order;
  int best = INT32_MAX;
  long budget = 200000;
  std::unordered_map<Mask, int> seen;
  Mask done;
  std::function<void(int, int)> dfs = [&](int live, int peak) {
    if (peak >= best || --budget < 0) return;
    if ((int)order.size() == nops) {
      best = peak;
      best_order = order;
      return;
    }
    auto it = seen.find(done);
    if (it != seen.end() && it->second <= peak) return;
    seen[done] = peak;
    for (int i = 0; i < nops; ++i) {
      if (done[i]) continue;
      bool ready = true;
      for (int d : deps[i]) ready &= (bool)done[d];
      if (!ready) continue;
      const BOp& o = r.ops[i];
      const bool mat = !r.is_vec[o.dst];
      bool inplace = false;
      for (int v : inplace_operands(o, ab))
        inplace |= !r.is_vec[v] && uses[v] == 1 && !keep[v] &&
                   std::count(reads[i].begin(), reads[i].end(), v) == 1;
      const int during = live + (mat && !inplace ? 1 : 0);
      int after = live;
      if (mat && (uses[o.dst] > 0 || keep[o.dst])) after += 1;
      for (int v : reads[i])
        if (--uses[v] == 0 && !keep[v]) after -= 1;
      done[i] = true;
      order.push_back(i);
      dfs(after, std::max(peak, during));
      order.pop_back();
      done[i] = false;
      for (int v : reads[i]) ++uses[v];
      if (budget < 0) return;
    }
  };
  dfs(live0, live0);
  if ((int)best_order.size() != nops) return;
  std::vector<BOp> ops(nops);
  for (int i = 0; i < nops; ++i) ops[i] = r.ops[best_order[i]];
  r.ops.swap(ops);
}

// The search is deterministic in the recorded program, so its result is
// memoised (repeated launches of the same run re-record the same program).
void schedule_min_live_cached(Rec& r, const std::vector<int>& pinned,
                              const std::vector<std::pair<int, int>>& carried, bool ab) {
  static std::mutex mu;
  static std::unordered_map<std::string, std::vector<BOp>> cache;
  std::string key(reinterpret_cast<const char*>(r.ops.data()), r.ops.size() * sizeof(BOp));
  key.push_back(ab ? 'b' : 'c');
  for (int v : pinned) key.append(reinterpret_cast<const char*>(&v), sizeof v);
  for (auto& pr : carried) {
    key.append(reinterpret_cast<const char*>(&pr.first), sizeof pr.first);
    key.append(reinterpret_cast<const char*>(&pr.second), sizeof pr.second);
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      r.ops = it->second;
      return;
    }
  }
  schedule_min_live(r, pinned, carried, ab);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() < 256) cache.emplace(std::move(key), r.ops);
}

// Linear-scan assignment of virtual registers to shared-memory slots.
//  * pinned: live for the whole run (A, b);
//  * carried (in, out): `in` holds the state at the start of an iteration and
//    dies at its last use; `out` (its next value) is live from its definition to
//    the end and takes `in`'s slot when that is free -- no copy needed.
struct Alloc {
  std::vector<int16_t> phys;
  int nmat = 0, nvec = 0;
};

Alloc assign(const Rec& r, const std::vector<int>& pinned,
             const std::vector<std::pair<int, int>>& carried, bool ab) {
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
  std::vector<int> out_of(nv, -1);  // out -> in
  for (auto& pr : carried) {
    last[pr.second] = INT32_MAX;
    out_of[pr.second] = pr.first;
  }
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
  auto release = [&](int v) {
    if (v >= 0 && al.phys[v] >= 0 && last[v] != INT32_MAX && last[v] != -2) {
      (r.is_vec[v] ? free_v : free_m).push_back(al.phys[v]);
      last[v] = -2;
    }
  };
  for (int p : pinned) al.phys[p] = (int16_t)take(r.is_vec[p]);
  for (auto& pr : carried) al.phys[pr.first] = (int16_t)take(r.is_vec[pr.first]);
  for (auto& pr : carried)  // a carried input never read this iteration is free at once
    if (last[pr.first] == -1) release(pr.first);
  for (int i = 0; i < (int)r.ops.size(); ++i) {
    const BOp& o = r.ops[i];
    const bool vec = r.is_vec[o.dst];
    if (al.phys[o.dst] < 0) {
      // in place over an operand that dies here (the carried input first)
      // (preference: the carried input itself, then an operand that sits in the
      // carried input's slot -- the next value lands where the next iteration
      // reads it, so no carry copy is needed -- then the first candidate)
      int reuse = -1;
      const int home = out_of[o.dst] >= 0 ? al.phys[out_of[o.dst]] : -1;
      auto rank = [&](int v) { return v == out_of[o.dst] ? 2 : (home >= 0 && al.phys[v] == home); };
      for (int v : inplace_operands(o, ab)) {
        if (v < 0 || r.is_vec[v] != vec || al.phys[v] < 0 || last[v] != i) continue;
        if (reuse < 0 || rank(v) > rank(reuse)) reuse = v;
      }
      if (reuse >= 0) {
        al.phys[o.dst] = al.phys[reuse];
        last[reuse] = -2;  // its slot now belongs to dst
      }
    }
    if (al.phys[o.dst] < 0) {
      const int in = out_of[o.dst];
      auto& fl = vec ? free_v : free_m;
      auto it = in >= 0 ? std::find(fl.begin(), fl.end(), (int)al.phys[in]) : fl.end();
      if (it != fl.end()) {
        al.phys[o.dst] = (int16_t)*it;
        fl.erase(it);
      } else {
        al.phys[o.dst] = (int16_t)take(vec);
      }
    }
    auto rel_if_last = [&](int v) {
      if (v >= 0 && last[v] == i) release(v);
    };
    rel_if_last(o.a);
    rel_if_last(o.b);
    rel_if_last(o.c);
    if (o.kind == OP_LIN)
      for (int j = 0; j < o.nterms; ++j) rel_if_last(o.t[j]);
    if (last[o.dst] == -1) release(o.dst);  // never read
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
  const double* p_in;  // carried state in (may equal the outputs)
  const double* f_in;
  const double* theta_in;
  double* p_io;  // carried state out
  double* f_io;
  double* theta_io;
  const DOp* ops;
  const double* cst;
  int ncst;
  int nops;
  int nmat;
  int nvec;
  int n;
  int iters;
  int64_t batch;
  int has_load;            // the program streams S^-1 / B in (OP_LOAD)
  int last_load;           // index of the last OP_LOAD: the next prefetch is issued after it
  long long* prof;         // per-op cycle totals of CTA 0 (diagnostics; usually null)
  int sA, sG, sF, sT, sb;  // slots of A, the carried inputs, b
  int sP, sB;              // resident splitting S^-1, B (-1: streamed by OP_LOAD)
  // inputs arriving by chunks of systems (host->device copies in flight): the
  // CTA waits for chunk_ready[sys / chunk] >= epoch before loading system sys
  // and counts finished systems in chunk_done[sys / chunk] (may be null)
  const unsigned* chunk_ready;
  unsigned* chunk_done;
  unsigned epoch;
  int64_t chunk;
  int rG, rF, rT;          // slots of the carried outputs (copied back when different)
  // dynamic system scheduling (one-CTA-per-system kernel): CTA b starts with
  // system b and claims gridDim.x + atomicAdd(sys_counter, 1) next (zeroed per
  // launch); null = static stride gridDim.x
  unsigned long long* sys_counter;
};

template <int NP>
struct Geo {
  static constexpr int SLOT = NP * NP;
#ifndef SI_RESIDENT_WARPS32
#define SI_RESIDENT_WARPS32 4
#endif
#ifndef SI_RESIDENT_WARPS64
#define SI_RESIDENT_WARPS64 16
#endif
  // NP=32: four warps with 16x16 warp tiles (2x2 DMMA tiles), four CTAs per
  // SM (registers: 122 per thread) -- 16 warps, 4 per SM sub-partition, all
  // CTAs alike.  Measured at C2 with dynamic system claims (tools/c2time.py):
  // 4 warps x 4 CTAs 2746 iters/s, x 5 CTAs (95 registers) 2722, x 3 CTAs
  // 2603; 2 warps of 32x16 x 5 CTAs 2680, x 4 CTAs 2625; 1 warp of 32x32
  // 1866.  NP=64 runs one CTA per SM: 16 warps hide latency.
  static constexpr int WARPS = NP == 32 ? SI_RESIDENT_WARPS32 : SI_RESIDENT_WARPS64;
  static constexpr int THREADS = WARPS * 32;
  // warp tile: a single warp owns the whole NP x NP product; otherwise the
  // warps form a (WARPS/2) x 2 grid
  static constexpr int WROWS = WARPS == 1 ? NP : NP / (WARPS / 2);
  static constexpr int WCOLS = WARPS == 1 ? NP : NP / 2;
  static constexpr int MT = WROWS / 8, NT = WCOLS / 8;
  // 16-byte chunk swizzle of row r: a distinct even value for the four rows
  // of a fragment (conflict-free 8-byte fragment loads), with rows 2q and 2q+1
  // in opposite halves of the 128-byte bank window (conflict-free 16-byte
  // accumulator stores)
  __device__ static __forceinline__ int swz(int r) { return ((r & 1) << 2) | (r & 2); }
  // element (r, c) of a slot
  __device__ static __forceinline__ int idx(int r, int c) {
    return r * NP + ((((c >> 1) ^ swz(r))) << 1) + (c & 1);
  }
  // logical column of the element stored at position (r, p)
  __device__ static __forceinline__ int col_at(int r, int p) {
    return ((((p >> 1) ^ swz(r))) << 1) + (p & 1);
  }
};

// Inputs of a gated launch are written by copy engines while the kernel runs:
// they are read with coherent (relaxed, gpu-scope) loads after the chunk flag
// was acquired -- the non-coherent __ldg path is only defined for data that
// stays read-only for the kernel's whole lifetime (the ungated case).
__device__ __forceinline__ double2 ld_in2(const double2* p, bool coherent) {
  if (coherent) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
  }
  return __ldg(p);
}
__device__ __forceinline__ double ld_in(const double* p, bool coherent) {
  if (coherent) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
  }
  return __ldg(p);
}

template <int NP>
__device__ void load_mat(double* dst, const double* __restrict__ src, int n,
                         bool coherent = false) {
  using G = Geo<NP>;
  if (n == NP) {
    // all of this thread's 16-byte loads in flight before the first store
    constexpr int PER = NP * NP / 2 / G::THREADS;
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2 v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = ld_in2(s2 + threadIdx.x + j * G::THREADS, coherent);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * G::THREADS;
      const int r = (2 * i) / NP, c = (2 * i) % NP;  // c even: one swizzled chunk
      *reinterpret_cast<double2*>(dst + G::idx(r, c)) = v[j];
    }
  } else {
    for (int i = threadIdx.x; i < NP * NP; i += G::THREADS) {
      const int r = i / NP, c = i % NP;
      dst[G::idx(r, c)] = (r < n && c < n) ? ld_in(src + r * n + c, coherent) : 0.0;
    }
  }
}

template <int NP>
__device__ void store_mat(double* __restrict__ dst, const double* src, int n) {
  using G = Geo<NP>;
  if (n == NP) {
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int i = threadIdx.x; i < NP * NP / 2; i += G::THREADS) {
      const int r = (2 * i) / NP, c = (2 * i) % NP;
      d2[i] = *reinterpret_cast<const double2*>(src + G::idx(r, c));
    }
  } else {
    for (int i = threadIdx.x; i < n * n; i += G::THREADS) dst[i] = src[G::idx(i / n, i % n)];
  }
}

__device__ __forceinline__ unsigned ld_acquire_u32_b(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t resident_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Sign flip on the integer pipe: the FP64 pipe is shared with DMMA.
__device__ __forceinline__ double flip(double x) {
  return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x));
}

// One NP x NP x NP product of a recorded op by the whole CTA.  MODE: 0 = A@B,
// 1 = I - A@B, 2 = A@B + C, 3 = generic alpha/beta/diag epilogue.
// The epilogue terms of modes 1 and 2 enter through the accumulator (C, or
// -I with the result negated), so those products issue no FP64-pipe
// instruction besides the DMMAs: on sm_100 the FP64 ALU shares its dispatch
// with the DMMA pipe, and epilogue adds stalled behind the other CTAs' DMMAs.
template <int NP, int MODE>
__device__ __forceinline__ void gemm_op(const double* A, const double* B, const double* C,
                                        double* D, const double* cst, int n, int warp, int g,
                                        int t, bool prebar) {
  using G = Geo<NP>;
  const int r0 = (warp >> 1) * G::WROWS, c0 = (warp & 1) * G::WCOLS;
  double acc[G::MT][G::NT][2];
#pragma unroll
  for (int mi = 0; mi < G::MT; ++mi)
#pragma unroll
    for (int ni = 0; ni < G::NT; ++ni) {
      const int row = r0 + mi * 8 + g, col = c0 + ni * 8 + 2 * t;
      if (MODE == 2) {
        const double2 cv = *reinterpret_cast<const double2*>(C + G::idx(row, col));
        acc[mi][ni][0] = cv.x;
        acc[mi][ni][1] = cv.y;
      } else if (MODE == 1) {
        acc[mi][ni][0] = (row == col && row < n) ? -1.0 : 0.0;
        acc[mi][ni][1] = (row == col + 1 && row < n) ? -1.0 : 0.0;
      } else {
        acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      }
    }
  double af[2][G::MT], bf[2][G::NT];
#pragma unroll
  for (int mi = 0; mi < G::MT; ++mi) af[0][mi] = A[G::idx(r0 + mi * 8 + g, t)];
#pragma unroll
  for (int ni = 0; ni < G::NT; ++ni) bf[0][ni] = B[G::idx(t, c0 + ni * 8 + g)];
#pragma unroll
  for (int kk = 0; kk < NP; kk += 4) {
    const int cur = (kk >> 2) & 1, nxt = cur ^ 1;
    if (kk + 4 < NP) {  // fragments of the next k-step in flight during this one
#pragma unroll
      for (int mi = 0; mi < G::MT; ++mi) af[nxt][mi] = A[G::idx(r0 + mi * 8 + g, kk + 4 + t)];
#pragma unroll
      for (int ni = 0; ni < G::NT; ++ni) bf[nxt][ni] = B[G::idx(kk + 4 + t, c0 + ni * 8 + g)];
    }
#pragma unroll
    for (int mi = 0; mi < G::MT; ++mi)
#pragma unroll
      for (int ni = 0; ni < G::NT; ++ni)
        dmma(acc[mi][ni][0], acc[mi][ni][1], af[cur][mi], bf[cur][ni]);
  }
  if (prebar) __syncthreads();  // D is A's or B's slot: every warp is done reading it
#pragma unroll
  for (int mi = 0; mi < G::MT; ++mi)
#pragma unroll
    for (int ni = 0; ni < G::NT; ++ni) {
      const int row = r0 + mi * 8 + g, col = c0 + ni * 8 + 2 * t;
      double v0 = acc[mi][ni][0], v1 = acc[mi][ni][1];
      if (MODE == 1) {
        v0 = flip(v0);
        v1 = flip(v1);
      } else if (MODE == 3) {
        double2 cv = make_double2(0.0, 0.0);
        if (C) cv = *reinterpret_cast<const double2*>(C + G::idx(row, col));
        v0 = epi(v0, cst[0], cst[1], cv.x);
        v1 = epi(v1, cst[0], cst[1], cv.y);
        if (cst[2] != 0.0 && row < n) {
          if (row == col) v0 = __dadd_rn(v0, cst[2]);
          if (row == col + 1) v1 = __dadd_rn(v1, cst[2]);
        }
      }
      *reinterpret_cast<double2*>(D + G::idx(row, col)) = make_double2(v0, v1);
    }
}

// The op program either comes from shared memory (interpreted: any recipe)
// or is baked in at compile time (FX::kFixed: the config-2 recipe, generated
// into resident_fixed_c2.inc by tools/gen_resident_fixed.py): then every op's
// kind, mode, slots and barrier flag are constants, the op loop is straight-
// line code, and no op is decoded or branched on at run time.
struct NoFixed {
  static constexpr bool kFixed = false;  // (ops / nops are only read under if constexpr)
};

#if __has_include("resident_fixed_c2.inc")
// BASELINE config 2's program (n = 32, rates (2, 3), order_n = 2)
struct FixedC2 {
#include "resident_fixed_c2.inc"
};
#define SI_HAVE_FIXED_C2 1
#endif
#if __has_include("resident_fixed_c1.inc")
// BASELINE config 1's program (one 64 x 64 system, NS order 3, 8-CTA cluster)
struct FixedC1 {
#include "resident_fixed_c1.inc"
};
#define SI_HAVE_FIXED_C1 1
#endif

template <class F, int... K>
__device__ __forceinline__ void static_for(F&& f, std::integer_sequence<int, K...>) {
  (f(std::integral_constant<int, K>{}), ...);
}

template <int NP, class FX = NoFixed>
// 32 x 32 systems: four CTAs of four warps per SM (<= 128 registers per
// thread; five fit in shared memory but measured slower, see Geo)
#ifndef SI_RESIDENT_MINB32
#define SI_RESIDENT_MINB32 4
#endif
__global__ void __launch_bounds__(Geo<NP>::THREADS, NP == 32 ? SI_RESIDENT_MINB32 : 1)
    resident_kernel(BatchArgs p) {
  using G = Geo<NP>;
  extern __shared__ double sm[];
  // dynamic shared memory: [matrix slots][vector slots][program][constants]
  DOp* prog = reinterpret_cast<DOp*>(sm + (size_t)p.nmat * G::SLOT + (size_t)p.nvec * NP);
  double* cst = reinterpret_cast<double*>(prog + p.nops);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n = p.n;
  const int64_t nn = (int64_t)n * n;
  auto mslot = [&](int s) { return sm + (size_t)s * G::SLOT; };
  __shared__ long long prof_acc[kMaxOps];  // SI_RESIDENT_PROF diagnostics (CTA 0, thread 0)
  long long prof_last = clock64();
  if (p.prof && threadIdx.x == 0)
    for (int k = 0; k < kMaxOps; ++k) prof_acc[k] = 0;
  auto vslot = [&](int s) { return sm + (size_t)p.nmat * G::SLOT + (size_t)s * NP; };
  for (int i = threadIdx.x; i < p.nops * (int)sizeof(DOp) / 16; i += G::THREADS)
    reinterpret_cast<int4*>(prog)[i] = reinterpret_cast<const int4*>(p.ops)[i];
  for (int i = threadIdx.x; i < p.ncst; i += G::THREADS) cst[i] = p.cst[i];
  __syncthreads();

  constexpr int PFD = NP * NP / 2 / G::THREADS > 0 ? NP * NP / 2 / G::THREADS : 1;
  double2 pf_p[PFD], pf_b[PFD];
  // Systems are claimed dynamically: the CTAs of an SM sub-partition holding
  // more warps than another run slower, and a static stride would leave the
  // whole launch waiting on them.  Which CTA runs a system does not change its
  // result (same program, same order).
  __shared__ int64_t s_next;
  int64_t sys = blockIdx.x;
  for (bool first = true; sys < p.batch; first = false) {
    if (threadIdx.x == 0)
      s_next = p.sys_counter ? (int64_t)gridDim.x + (int64_t)atomicAdd(p.sys_counter, 1ull)
                             : sys + gridDim.x;
    if (p.chunk_ready) {  // this system's inputs may still be copying
      if (threadIdx.x == 0) {
        const unsigned* f = p.chunk_ready + sys / p.chunk;
        const uint64_t t0 = resident_timer_ns();
        while ((int)(ld_acquire_u32_b(f) - p.epoch) < 0) {
          __nanosleep(128);
          if (resident_timer_ns() - t0 > 60ull * 1000000000ull) __trap();
        }
      }
      __syncthreads();
    }
    const bool gated = p.chunk_ready != nullptr;
    load_mat<NP>(mslot(p.sA), p.a + sys * nn, n, gated);
    if (p.sP >= 0) load_mat<NP>(mslot(p.sP), p.precond + sys * nn, n, gated);
    if (p.sB >= 0) load_mat<NP>(mslot(p.sB), p.residual + sys * nn, n, gated);
    load_mat<NP>(mslot(p.sG), p.p_in + sys * nn, n, gated);
    load_mat<NP>(mslot(p.sF), p.f_in + sys * nn, n, gated);
    if (threadIdx.x < NP) {
      vslot(p.sT)[threadIdx.x] =
          threadIdx.x < n ? ld_in(p.theta_in + sys * n + threadIdx.x, gated) : 0.0;
      vslot(p.sb)[threadIdx.x] = threadIdx.x < n ? ld_in(p.b + sys * n + threadIdx.x, gated) : 0.0;
    }
    __syncthreads();
    const int64_t nxt = s_next;  // written by thread 0 before the barrier above
    // S^-1 and B are streamed in every iteration through registers: the global
    // loads for the next iteration (or the next system) are issued right after
    // the last LOAD op consumed the previous ones, so their latency hides behind
    // the rest of the iteration (full-size systems only)
    constexpr int PF = NP * NP / 2 / G::THREADS;
    const bool prefetch = p.has_load && n == NP && PF >= 1;
    auto issue = [&](int64_t s) {
      const double2* sp2 = reinterpret_cast<const double2*>(p.precond + s * nn);
      const double2* sb2 = reinterpret_cast<const double2*>(p.residual + s * nn);
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        pf_p[j] = ld_in2(sp2 + threadIdx.x + j * G::THREADS, gated);
        pf_b[j] = ld_in2(sb2 + threadIdx.x + j * G::THREADS, gated);
      }
    };
    if (prefetch && (first || p.chunk_ready)) issue(sys);
    // one op of the program; `o` is a compile-time constant on the fixed path
    auto exec = [&](const DOp& o, int k, int it) {
        const double* oc = cst + o.cidx;
        if (o.kind == OP_LOAD && prefetch) {
          double* dst = mslot(o.dst);
#pragma unroll
          for (int j = 0; j < PF; ++j) {
            const int i = threadIdx.x + j * G::THREADS;
            const int r = (2 * i) / NP, c = (2 * i) % NP;
            *reinterpret_cast<double2*>(dst + G::idx(r, c)) = o.mode ? pf_b[j] : pf_p[j];
          }
          if (k == p.last_load) {
            if (it + 1 < p.iters)
              issue(sys);
            else if (nxt < p.batch && !p.chunk_ready)  // gated: at system start
              issue(nxt);
          }
        } else if (o.kind == OP_GEMM) {
          const double* A = mslot(o.a);
          const double* B = mslot(o.b);
          const double* C = o.c >= 0 ? mslot(o.c) : nullptr;
          double* D = mslot(o.dst);
          const bool pb = o.prebar != 0;
          // the DAG's epilogues are "X@Y", "I - X@Y" and "X@Y + Z": specialised,
          // anything else goes through the generic path
          switch (o.mode) {
            case 0: gemm_op<NP, 0>(A, B, C, D, oc, n, warp, g, t, pb); break;
            case 1: gemm_op<NP, 1>(A, B, C, D, oc, n, warp, g, t, pb); break;
            case 2: gemm_op<NP, 2>(A, B, C, D, oc, n, warp, g, t, pb); break;
            default: gemm_op<NP, 3>(A, B, C, D, oc, n, warp, g, t, pb); break;
          }
        } else if (o.kind == OP_GEMV) {
          // On the DMMA pipe, not the FP64 ALU: x becomes column 0 of an 8-wide B
          // fragment (zeros elsewhere).  A DFMA + shuffle-tree GEMV contends with
          // the other resident CTAs' DMMAs and was 2.5x slower than a full GEMM op.
          // Each warp takes its 8-row tiles side by side with K split over 4
          // accumulator sets: the dependent DMMA chains are NP/16 deep and
          // interleaved (GEMVs are latency, not throughput).
          constexpr int RTW = (NP / 8 + G::WARPS - 1) / G::WARPS;
          const double* A = mslot(o.a);
          const double* x = vslot(o.b);
          double acc[RTW][4][2] = {};
#pragma unroll
          for (int kk = 0; kk < NP; kk += 4) {
            const double bf = g == 0 ? x[kk + t] : 0.0;
#pragma unroll
            for (int j = 0; j < RTW; ++j) {
              const int rt = warp + j * G::WARPS;
              if (rt < NP / 8) {
                const double af = A[G::idx(rt * 8 + g, kk + t)];
                dmma(acc[j][(kk >> 2) & 3][0], acc[j][(kk >> 2) & 3][1], af, bf);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < RTW; ++j) {
            const int rt = warp + j * G::WARPS;
            if (rt < NP / 8 && t == 0) {  // lane (g, 0) holds row rt*8 + g, column 0
              const int row = rt * 8 + g;
              const double s = __dadd_rn(__dadd_rn(acc[j][0][0], acc[j][1][0]),
                                         __dadd_rn(acc[j][2][0], acc[j][3][0]));
              const double cv = o.c >= 0 ? vslot(o.c)[row] : 0.0;
              double v;
              if (o.mode == 1)
                v = __dsub_rn(s, cv);  // A x - c
              else if (o.mode == 2)
                v = __dsub_rn(cv, s);  // c - A x
              else
                v = epi(s, oc[0], oc[1], cv);
              vslot(o.dst)[row] = v;
            }
          }
        } else if (o.kind == OP_LOAD) {
          load_mat<NP>(mslot(o.dst), (o.mode ? p.residual : p.precond) + sys * nn, n, gated);
        } else if (o.mode) {  // LIN over vectors
          if (threadIdx.x < NP) {
            double acc = 0.0;
            for (int j = 0; j < o.nterms; ++j) {
              // (the term list is read from shared memory on the interpreted
              // path: indexing a register copy of `o` with a runtime j would
              // put it in local memory)
              const int tj = FX::kFixed ? o.t[j] : prog[k].t[j];
              const double xv = vslot(tj)[threadIdx.x];
              acc = __dadd_rn(acc, oc[1 + j] == 1.0 ? xv : __dmul_rn(oc[1 + j], xv));
            }
            vslot(o.dst)[threadIdx.x] = acc;
          }
        } else {  // LIN over matrices
          double* D = mslot(o.dst);
          for (int i = threadIdx.x; i < NP * NP; i += G::THREADS) {
            const int r = i / NP;
            const int c = G::col_at(r, i % NP);
            double acc = (r == c && r < n) ? oc[0] : 0.0;
            for (int j = 0; j < o.nterms; ++j) {
              const int tj = FX::kFixed ? o.t[j] : prog[k].t[j];
              const double xv = mslot(tj)[i];
              acc = __dadd_rn(acc, oc[1 + j] == 1.0 ? xv : __dmul_rn(oc[1 + j], xv));
            }
            D[i] = acc;
          }
        }
        if (o.sync) __syncthreads();  // elided when the next op is independent
        if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) {  // SI_RESIDENT_PROF diagnostics
          const long long now = clock64();
          prof_acc[k] += now - prof_last;
          prof_last = now;
        }
    };
    for (int it = 0; it < p.iters; ++it) {
      if constexpr (FX::kFixed) {
        static_for(
            [&](auto kc) {
              constexpr int k = decltype(kc)::value;
              constexpr DOp o = FX::ops[k];
              exec(o, k, it);
            },
            std::make_integer_sequence<int, FX::nops>{});
      } else {
        for (int k = 0; k < p.nops; ++k) {
          const DOp o = prog[k];
          exec(o, k, it);
        }
      }
      // carry the state where the allocator could not place it in place
      if (p.rG != p.sG || p.rF != p.sF) {
        for (int i = threadIdx.x; i < NP * NP; i += G::THREADS) {
          if (p.rG != p.sG) mslot(p.sG)[i] = mslot(p.rG)[i];
          if (p.rF != p.sF) mslot(p.sF)[i] = mslot(p.rF)[i];
        }
      }
      if (p.rT != p.sT && threadIdx.x < NP) vslot(p.sT)[threadIdx.x] = vslot(p.rT)[threadIdx.x];
      __syncthreads();
    }
    store_mat<NP>(p.p_io + sys * nn, mslot(p.sG), n);
    store_mat<NP>(p.f_io + sys * nn, mslot(p.sF), n);
    if (threadIdx.x < n) p.theta_io[sys * n + threadIdx.x] = vslot(p.sT)[threadIdx.x];
    __syncthreads();
    if (p.chunk_done && threadIdx.x == 0) {  // outputs of sys visible, then counted
      __threadfence_system();
      atomicAdd(p.chunk_done + sys / p.chunk, 1u);
    }
    sys = nxt;
  }
  if (p.prof && blockIdx.x == 0 && threadIdx.x == 0)
    for (int k = 0; k < p.nops; ++k) p.prof[k] = prof_acc[k];
}

// ---------------------------------------------------------------- clusters
// Latency-bound small batches (config 1: ONE 64 x 64 system): a thread-block
// cluster of CL CTAs (CL SMs) works on one system.  Every CTA keeps a full
// copy of every slot but computes only its block of NP/CL rows of each op;
// results that a later op reads in full (right operands of products, the x of
// a GEMV, loop-carried ones included) are also stored into the peers' copies
// through distributed shared memory, and cluster barriers order those
// exchanges (flags decided on the host, cluster_flags()).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t peer_addr(const double* local, unsigned cta) {
  const uint32_t la = static_cast<uint32_t>(__cvta_generic_to_shared(local));
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(cta));
  return ra;
}
__device__ __forceinline__ void st_peer2(const double* local, unsigned cta, double x, double y) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(peer_addr(local, cta)), "d"(x),
               "d"(y)
               : "memory");
}
__device__ __forceinline__ void st_peer1(const double* local, unsigned cta, double x) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(peer_addr(local, cta)), "d"(x) : "memory");
}

constexpr int kClusterThreads = 256;  // 8 warps per CTA
constexpr uint8_t kSyncCta = 1, kSyncCluster = 2, kBcast = 4;

// Rows [rbase, rbase + 64/CL) of one 64 x 64 x 64 product, 8 warps.
template <int CL, int MODE>
__device__ __forceinline__ void gemm_rows(const double* A, const double* B, const double* C,
                                          double* D, const double* cst, int n, int warp, int g,
                                          int t, int rbase, bool bcast, unsigned rank) {
  using G = Geo<64>;
  constexpr int RT = 64 / CL / 8;             // 8-row tiles per CTA
  constexpr int NTW = RT >= 2 ? 2 : 1;        // column tiles per warp
  constexpr int CG = 8 / NTW, RG = 8 / CG;    // warp grid
  constexpr int MTW = RT / RG;                // row tiles per warp
  const int r0 = rbase + (warp / CG) * MTW * 8, c0 = (warp % CG) * NTW * 8;
  // KS accumulator sets take the k-steps in turn (k-step s into set s % KS)
  // and are summed in a fixed order at the end: with one 8 x 8 tile per warp
  // (8-CTA clusters) the 16 dependent DMMAs of a single chain (26 cycles
  // each) would set the op's latency
#ifndef SI_CLUSTER_KS
#define SI_CLUSTER_KS 4
#endif
  constexpr int KS = MTW * NTW == 1 ? SI_CLUSTER_KS : 1;
  static_assert(KS == 1 || KS == 4, "k-step accumulator sets: 1 or 4");
  double acc[MTW][NTW][2];
  double ex[KS > 1 ? KS - 1 : 1][2] = {};
#pragma unroll
  for (int mi = 0; mi < MTW; ++mi)
#pragma unroll
    for (int ni = 0; ni < NTW; ++ni) {
      const int row = r0 + mi * 8 + g, col = c0 + ni * 8 + 2 * t;
      if (MODE == 2) {
        const double2 cv = *reinterpret_cast<const double2*>(C + G::idx(row, col));
        acc[mi][ni][0] = cv.x;
        acc[mi][ni][1] = cv.y;
      } else if (MODE == 1) {
        acc[mi][ni][0] = (row == col && row < n) ? -1.0 : 0.0;
        acc[mi][ni][1] = (row == col + 1 && row < n) ? -1.0 : 0.0;
      } else {
        acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      }
    }
  double af[2][MTW], bf[2][NTW];
#pragma unroll
  for (int mi = 0; mi < MTW; ++mi) af[0][mi] = A[G::idx(r0 + mi * 8 + g, t)];
#pragma unroll
  for (int ni = 0; ni < NTW; ++ni) bf[0][ni] = B[G::idx(t, c0 + ni * 8 + g)];
#pragma unroll
  for (int kk = 0; kk < 64; kk += 4) {
    const int cur = (kk >> 2) & 1, nxt = cur ^ 1;
    if (kk + 4 < 64) {
#pragma unroll
      for (int mi = 0; mi < MTW; ++mi) af[nxt][mi] = A[G::idx(r0 + mi * 8 + g, kk + 4 + t)];
#pragma unroll
      for (int ni = 0; ni < NTW; ++ni) bf[nxt][ni] = B[G::idx(kk + 4 + t, c0 + ni * 8 + g)];
    }
    const int set = (kk >> 2) % KS;
    if (KS > 1 && set > 0) {
      dmma(ex[set - 1][0], ex[set - 1][1], af[cur][0], bf[cur][0]);
      continue;
    }
#pragma unroll
    for (int mi = 0; mi < MTW; ++mi)
#pragma unroll
      for (int ni = 0; ni < NTW; ++ni)
        dmma(acc[mi][ni][0], acc[mi][ni][1], af[cur][mi], bf[cur][ni]);
  }
  if constexpr (KS == 4) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      acc[0][0][h] = __dadd_rn(__dadd_rn(acc[0][0][h], ex[0][h]), __dadd_rn(ex[1][h], ex[2][h]));
  }
#pragma unroll
  for (int mi = 0; mi < MTW; ++mi)
#pragma unroll
    for (int ni = 0; ni < NTW; ++ni) {
      const int row = r0 + mi * 8 + g, col = c0 + ni * 8 + 2 * t;
      double v0 = acc[mi][ni][0], v1 = acc[mi][ni][1];
      if (MODE == 1) {
        v0 = flip(v0);
        v1 = flip(v1);
      } else if (MODE == 3) {
        double2 cv = make_double2(0.0, 0.0);
        if (C) cv = *reinterpret_cast<const double2*>(C + G::idx(row, col));
        v0 = epi(v0, cst[0], cst[1], cv.x);
        v1 = epi(v1, cst[0], cst[1], cv.y);
        if (cst[2] != 0.0 && row < n) {
          if (row == col) v0 = __dadd_rn(v0, cst[2]);
          if (row == col + 1) v1 = __dadd_rn(v1, cst[2]);
        }
      }
      double* dp = D + G::idx(row, col);
      *reinterpret_cast<double2*>(dp) = make_double2(v0, v1);
      if (bcast)
#pragma unroll
        for (unsigned q = 0; q < CL; ++q)
          if (q != rank) st_peer2(dp, q, v0, v1);
    }
}

template <int CL, class FX = NoFixed>
__global__ void __launch_bounds__(kClusterThreads, 1) resident_cluster_kernel(BatchArgs p) {
  constexpr int NP = 64, RB = NP / CL, TH = kClusterThreads;
  using G = Geo<64>;
  extern __shared__ double sm[];
  DOp* prog = reinterpret_cast<DOp*>(sm + (size_t)p.nmat * G::SLOT + (size_t)p.nvec * NP);
  double* cst = reinterpret_cast<double*>(prog + p.nops);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n = p.n;
  const int64_t nn = (int64_t)n * n;
  const unsigned rank = cluster_rank();
  const int rbase = (int)rank * RB;
  auto mslot = [&](int s) { return sm + (size_t)s * G::SLOT; };
  auto vslot = [&](int s) { return sm + (size_t)p.nmat * G::SLOT + (size_t)s * NP; };
  auto load_full = [&](double* dst, const double* src) {
    for (int i = threadIdx.x; i < NP * NP; i += TH) {
      const int r = i / NP, c = i % NP;
      dst[G::idx(r, c)] = (r < n && c < n) ? src[r * n + c] : 0.0;
    }
  };
  for (int i = threadIdx.x; i < p.nops * (int)sizeof(DOp) / 16; i += TH)
    reinterpret_cast<int4*>(prog)[i] = reinterpret_cast<const int4*>(p.ops)[i];
  for (int i = threadIdx.x; i < p.ncst; i += TH) cst[i] = p.cst[i];
  __shared__ long long prof_acc[kMaxOps];  // SI_RESIDENT_PROF diagnostics (CTA 0, thread 0)
  if (p.prof && threadIdx.x == 0)
    for (int k = 0; k < kMaxOps; ++k) prof_acc[k] = 0;
  long long prof_last = clock64();

  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  for (int64_t sys = cid; sys < p.batch; sys += ncl) {
    load_full(mslot(p.sA), p.a + sys * nn);
    if (p.sP >= 0) load_full(mslot(p.sP), p.precond + sys * nn);
    if (p.sB >= 0) load_full(mslot(p.sB), p.residual + sys * nn);
    load_full(mslot(p.sG), p.p_in + sys * nn);
    load_full(mslot(p.sF), p.f_in + sys * nn);
    if (threadIdx.x < NP) {
      vslot(p.sT)[threadIdx.x] = threadIdx.x < n ? p.theta_in[sys * n + threadIdx.x] : 0.0;
      vslot(p.sb)[threadIdx.x] = threadIdx.x < n ? p.b[sys * n + threadIdx.x] : 0.0;
    }
    cluster_sync_all();  // every CTA of the cluster is running and loaded
    // one op; `o` is a compile-time constant on the fixed path (FX::kFixed)
    auto exec = [&](const DOp& o, int k) {
        const double* oc = cst + o.cidx;
        const bool bc = (o.sync & kBcast) != 0;
        if (o.kind == OP_GEMM) {
          const double* A = mslot(o.a);
          const double* B = mslot(o.b);
          const double* C = o.c >= 0 ? mslot(o.c) : nullptr;
          double* D = mslot(o.dst);
          switch (o.mode) {
            case 0: gemm_rows<CL, 0>(A, B, C, D, oc, n, warp, g, t, rbase, bc, rank); break;
            case 1: gemm_rows<CL, 1>(A, B, C, D, oc, n, warp, g, t, rbase, bc, rank); break;
            case 2: gemm_rows<CL, 2>(A, B, C, D, oc, n, warp, g, t, rbase, bc, rank); break;
            default: gemm_rows<CL, 3>(A, B, C, D, oc, n, warp, g, t, rbase, bc, rank); break;
          }
        } else if (o.kind == OP_GEMV) {
          if (warp < RB / 8) {
            const double* A = mslot(o.a);
            const double* x = vslot(o.b);
            const int r0 = rbase + warp * 8;
            // interleaved chains of dependent DMMAs (4: chains of 4)
            constexpr int GS = SI_CLUSTER_KS == 1 ? 2 : 4;
            double acc[4][2] = {};
#pragma unroll
            for (int kk = 0; kk < NP; kk += 4) {
              const double af = A[G::idx(r0 + g, kk + t)];
              const double bf = g == 0 ? x[kk + t] : 0.0;
              dmma(acc[(kk >> 2) % GS][0], acc[(kk >> 2) % GS][1], af, bf);
            }
            if (t == 0) {
              const int row = r0 + g;
              const double s = __dadd_rn(__dadd_rn(acc[0][0], acc[1][0]),
                                         __dadd_rn(acc[2][0], acc[3][0]));
              const double cv = o.c >= 0 ? vslot(o.c)[row] : 0.0;
              const double v = o.mode == 1   ? __dsub_rn(s, cv)
                               : o.mode == 2 ? __dsub_rn(cv, s)
                                             : epi(s, oc[0], oc[1], cv);
              double* dp = vslot(o.dst) + row;
              *dp = v;
              if (bc)
                for (unsigned q = 0; q < CL; ++q)
                  if (q != rank) st_peer1(dp, q, v);
            }
          }
        } else if (o.kind == OP_LOAD) {
          load_full(mslot(o.dst), (o.mode ? p.residual : p.precond) + sys * nn);
        } else if (o.mode) {  // LIN over vectors, own rows
          if (threadIdx.x < RB) {
            const int row = rbase + threadIdx.x;
            double acc = 0.0;
            for (int j = 0; j < o.nterms; ++j) {
              const double xv = vslot((FX::kFixed ? o.t[j] : prog[k].t[j]))[row];
              acc = __dadd_rn(acc, oc[1 + j] == 1.0 ? xv : __dmul_rn(oc[1 + j], xv));
            }
            double* dp = vslot(o.dst) + row;
            *dp = acc;
            if (bc)
              for (unsigned q = 0; q < CL; ++q)
                if (q != rank) st_peer1(dp, q, acc);
          }
        } else {  // LIN over matrices, own rows
          double* D = mslot(o.dst);
          for (int i = rbase * NP + threadIdx.x; i < (rbase + RB) * NP; i += TH) {
            const int r = i / NP;
            const int c = G::col_at(r, i % NP);
            double acc = (r == c && r < n) ? oc[0] : 0.0;
            for (int j = 0; j < o.nterms; ++j) {
              const double xv = mslot((FX::kFixed ? o.t[j] : prog[k].t[j]))[i];
              acc = __dadd_rn(acc, oc[1 + j] == 1.0 ? xv : __dmul_rn(oc[1 + j], xv));
            }
            D[i] = acc;
            if (bc)
              for (unsigned q = 0; q < CL; ++q)
                if (q != rank) st_peer1(D + i, q, acc);
          }
        }
        if (o.sync & kSyncCluster)
          cluster_sync_all();
        else if (o.sync & kSyncCta)
          __syncthreads();
        if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) {
          const long long now = clock64();
          prof_acc[k] += now - prof_last;
          prof_last = now;
        }
    };
    for (int it = 0; it < p.iters; ++it) {
      if constexpr (FX::kFixed) {
        static_for(
            [&](auto kc) {
              constexpr int k = decltype(kc)::value;
              constexpr DOp o = FX::ops[k];
              exec(o, k);
            },
            std::make_integer_sequence<int, FX::nops>{});
      } else {
        for (int k = 0; k < p.nops; ++k) {
          const DOp o = prog[k];
          exec(o, k);
        }
      }
      if (p.rG != p.sG || p.rF != p.sF || p.rT != p.sT) {  // carries (full local copies)
        cluster_sync_all();  // every broadcast into the carried outputs has landed
        for (int i = threadIdx.x; i < NP * NP; i += TH) {
          if (p.rG != p.sG) mslot(p.sG)[i] = mslot(p.rG)[i];
          if (p.rF != p.sF) mslot(p.sF)[i] = mslot(p.rF)[i];
        }
        if (p.rT != p.sT && threadIdx.x < NP) vslot(p.sT)[threadIdx.x] = vslot(p.rT)[threadIdx.x];
        cluster_sync_all();
      }
    }
    // own rows of the outputs
    for (int i = rbase * n + threadIdx.x; i < min(rbase + RB, n) * n; i += TH) {
      const int r = i / n, c = i % n;
      p.p_io[sys * nn + i] = mslot(p.sG)[G::idx(r, c)];
      p.f_io[sys * nn + i] = mslot(p.sF)[G::idx(r, c)];
    }
    if (threadIdx.x < RB && rbase + (int)threadIdx.x < n)
      p.theta_io[sys * n + rbase + threadIdx.x] = vslot(p.sT)[rbase + threadIdx.x];
    cluster_sync_all();  // peers are done with this system before slots are reloaded
  }
  if (p.prof && blockIdx.x == 0 && threadIdx.x == 0)
    for (int k = 0; k < p.nops; ++k) p.prof[k] = prof_acc[k];
}

// Barrier / exchange flags of a cluster program (ops already on physical
// slots; `vec_dst[k]`: op k writes a vector slot; `bcast[k]`: its result is
// read in full somewhere, so it goes to every peer's copy too).  Before op
// j+1: a cluster barrier when it reads in full a slot broadcast since the last
// cluster barrier, or broadcasts into a slot read in full / broadcast since
// then; otherwise a CTA barrier on the usual RAW / WAR / WAW rule.  The
// program is analysed as a loop (iteration i's tail against i+1's head).
std::vector<uint8_t> cluster_flags(const std::vector<BOp>& prog, const std::vector<bool>& pbc) {
  // The program repeats: analyse three copies and keep the middle one's flags,
  // whose windows already carry the previous iteration's tail (the first
  // iteration starts after a cluster barrier, a subset of that state).
  const size_t m0 = prog.size();
  std::vector<BOp> ops;
  std::vector<bool> bcast;
  for (int rep = 0; rep < 3; ++rep) {
    ops.insert(ops.end(), prog.begin(), prog.end());
    bcast.insert(bcast.end(), pbc.begin(), pbc.end());
  }
  const size_t m = ops.size();
  std::vector<uint8_t> fl(m, 0);
  auto key = [](int s, bool vec) { return vec ? 1000 + s : s; };
  struct Acc {
    std::vector<int> rloc, rfull;
    int w;
    bool full_write = false;  // OP_LOAD: every CTA writes all rows of its copy
  };
  std::vector<Acc> acc(m);
  for (size_t k = 0; k < m; ++k) {
    const BOp& o = ops[k];
    Acc& a = acc[k];
    const bool vdst = (o.kind == OP_GEMV) || (o.kind == OP_LIN && o.vec);
    a.w = key(o.dst, vdst);
    if (o.kind == OP_GEMM) {
      a.rloc = {key(o.a, false)};
      if (o.c >= 0) a.rloc.push_back(key(o.c, false));
      a.rfull = {key(o.b, false)};
    } else if (o.kind == OP_GEMV) {
      a.rloc = {key(o.a, false)};
      if (o.c >= 0) a.rloc.push_back(key(o.c, true));
      a.rfull = {key(o.b, true)};
    } else if (o.kind == OP_LIN) {
      for (int j = 0; j < o.nterms; ++j) a.rloc.push_back(key(o.t[j], o.vec));
    } else {
      a.full_write = true;
    }
  }
  auto in = [](const std::vector<int>& v, int s) { return std::find(v.begin(), v.end(), s) != v.end(); };
  std::vector<int> rdC, wrC, rdF, wrB, wrF;
  for (size_t k = 0; k < m; ++k) {
    const Acc& a = acc[k];
    if (k > 0) {
      bool clu = false, cta = false;
      for (int s : a.rfull) clu |= in(wrB, s);
      if (bcast[k]) clu |= in(rdF, a.w) || in(wrB, a.w) || in(wrF, a.w);
      for (int s : a.rloc) cta |= in(wrC, s);
      for (int s : a.rfull) cta |= in(wrC, s);
      cta |= in(rdC, a.w) || in(wrC, a.w);
      if (clu) {
        fl[k - 1] |= kSyncCluster;
        rdC.clear(); wrC.clear(); rdF.clear(); wrB.clear(); wrF.clear();
      } else if (cta) {
        fl[k - 1] |= kSyncCta;
        rdC.clear(); wrC.clear();
      }
    }
    rdC.insert(rdC.end(), a.rloc.begin(), a.rloc.end());
    rdC.insert(rdC.end(), a.rfull.begin(), a.rfull.end());
    rdF.insert(rdF.end(), a.rfull.begin(), a.rfull.end());
    wrC.push_back(a.w);
    if (bcast[k]) wrB.push_back(a.w);
    if (a.full_write) wrF.push_back(a.w);
  }
  std::vector<uint8_t> out(fl.begin() + m0, fl.begin() + 2 * m0);
  bool any = false;
  for (uint8_t f : out) any |= (f & kSyncCluster) != 0;
  if (!any && m0) out[m0 - 1] |= kSyncCluster;  // windows must not grow without bound
  for (size_t k = 0; k < m0; ++k)
    if (pbc[k]) out[k] |= kBcast;
  return out;
}

// SI_RESIDENT_FIXED=0: always interpret (A/B measurements; read once)
bool fixed_disabled() {
  static const bool off = [] {
    const char* v = std::getenv("SI_RESIDENT_FIXED");
    return v != nullptr && v[0] == '0';
  }();
  return off;
}

int num_sms_b() {
  int d = 0, n = 0;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  return n;
}

// Registers of a recorded iteration.
struct Recipe {
  Rec r;
  int A, G, F, T, bv;
  int P = -1, B = -1;  // resident splitting (pinned) instead of per-iteration loads
  int gn = -1, fn = -1, tn = -1;
};

Recipe new_recipe() {
  Recipe q;
  q.A = q.r.fresh(false);
  q.G = q.r.fresh(false);
  q.F = q.r.fresh(false);
  q.T = q.r.fresh(true);
  q.bv = q.r.fresh(true);
  return q;
}

// plain Richardson with P_k = G (before the inversion update)
void record_plain(Recipe& q) {
  const int res = q.r.gemv(q.A, q.T, 1.0, q.bv, -1.0);  // A theta - b
  q.tn = q.r.gemv(q.G, res, -1.0, q.T, 1.0);            // theta - P resid
}

// theta' is only read by the next iteration: move its GEMV behind the first
// product, so that product overlaps both GEMVs (the residual GEMV runs while
// the product's other warps start; theta' runs while the next product does)
// instead of the GEMV pair forming a serial prologue.
void defer_theta_update(Recipe& q) {
  auto& ops = q.r.ops;
  int i1 = -1;
  for (int i = 0; i < (int)ops.size(); ++i)
    if (ops[i].dst == q.tn) i1 = i;
  if (i1 < 0) return;
  for (int j = i1 + 1; j < (int)ops.size(); ++j)
    if (ops[j].kind == OP_GEMM) {
      const BOp mv = ops[i1];
      ops.erase(ops.begin() + i1);
      ops.insert(ops.begin() + j, mv);  // now just after that product
      return;
    }
}

// The device program of a recipe: scheduled, slot-allocated, barrier flags,
// device encoding (host only; no CUDA call except the SM count for NP = 64).
struct Built {
  std::vector<BOp> ops;
  std::vector<DOp> dev_ops;
  std::vector<double> csts;
  Alloc al;
  int cl = 0;
  std::vector<uint8_t> cflags;
  size_t smem = 0;
  std::string blob;  // dev_ops + csts: what the kernel reads
};

template <int NP>
Built build_program(Recipe& q, int64_t batch, const ChunkGate* gate, int force_cl = -1) {
  using Gm = Geo<NP>;
  if ((int)q.r.ops.size() > kMaxOps) throw Error(kEInval, "resident program too long");

  std::vector<int> pinned = {q.A, q.bv};
  if (q.P >= 0) pinned.push_back(q.P);
  if (q.B >= 0) pinned.push_back(q.B);
  // products over their own A / B operand: one-CTA-per-system kernel only
  // (NP = 64 may run as a cluster, whose peers read broadcast copies)
  const bool ab = NP == 32;
  schedule_min_live_cached(q.r, pinned, {{q.G, q.gn}, {q.F, q.fn}, {q.T, q.tn}}, ab);
  Built bt;
  Alloc& al = bt.al;
  al = assign(q.r, pinned, {{q.G, q.gn}, {q.F, q.fn}, {q.T, q.tn}}, ab);
  std::vector<BOp>& ops = bt.ops;
  ops = q.r.ops;
  auto ph = [&](int v) -> int16_t { return v >= 0 ? al.phys[v] : (int16_t)-1; };
  for (BOp& o : ops) {
    o.dst = ph(o.dst);
    o.a = ph(o.a);
    o.b = ph(o.b);
    o.c = ph(o.c);
    if (o.kind == OP_LIN)
      for (int j = 0; j < o.nterms; ++j) o.t[j] = ph(o.t[j]);
  }
  // Barrier elision: op k+1 may start before op k has finished in every warp
  // when it neither reads a slot written since the last barrier (RAW) nor
  // writes a slot read or written since then (WAR / WAW).  Independent ops of
  // the DAG (e.g. Gamma_1 and the next part's first product) then overlap.
  {
    auto key = [&](const BOp& o, int s, bool vec) { return vec ? 1000 + s : s; };
    std::vector<int> rd, wr;
    auto hit = [](const std::vector<int>& v, int s) {
      return std::find(v.begin(), v.end(), s) != v.end();
    };
    for (size_t k = 0; k < ops.size(); ++k) {
      BOp& o = ops[k];
      std::vector<int> reads, writes;
      const bool vdst = (o.kind == OP_GEMV) || (o.kind == OP_LIN && o.vec);
      writes.push_back(key(o, o.dst, vdst));
      if (o.kind == OP_GEMM) {
        reads = {key(o, o.a, false), key(o, o.b, false)};
        if (o.c >= 0) reads.push_back(key(o, o.c, false));
      } else if (o.kind == OP_GEMV) {
        reads = {key(o, o.a, false), key(o, o.b, true)};
        if (o.c >= 0) reads.push_back(key(o, o.c, true));
      } else if (o.kind == OP_LIN) {
        for (int j = 0; j < o.nterms; ++j) reads.push_back(key(o, o.t[j], o.vec));
      }
      bool need = false;
      for (int s : reads) need |= hit(wr, s);
      for (int s : writes) need |= hit(wr, s) || hit(rd, s);
      if (k > 0) ops[k - 1].pad_ = need ? 1 : 0;  // barrier after the previous op
      if (need) {
        rd.clear();
        wr.clear();
      }
      rd.insert(rd.end(), reads.begin(), reads.end());
      wr.insert(wr.end(), writes.begin(), writes.end());
    }
    if (!ops.empty()) ops.back().pad_ = 1;  // end of iteration: carry copies follow
  }
  // Cluster mode (NP = 64, few systems: latency-bound on one SM each): one
  // cluster of `cl` CTAs per system.  SI_RESIDENT_CLUSTER = 0/2/4/8 overrides.
  int& cl = bt.cl;
  if (NP == 64) {
    const char* env = std::getenv("SI_RESIDENT_CLUSTER");
    if (force_cl >= 0) {
      cl = force_cl;  // (build tooling: no device to ask for its SM count)
    } else if (env) {
      cl = std::atoi(env);
      if (cl != 0 && cl != 2 && cl != 4 && cl != 8) cl = 0;
    } else if (batch * 8 <= num_sms_b()) {
      cl = 8;  // C1: 8-row blocks per SM, 192k vs 187k iters/s with 4 SMs
    } else if (batch * 4 <= num_sms_b()) {
      cl = 4;
    }
    if (gate && gate->ready) cl = 0;  // the chunk gate lives in the one-CTA kernel
  }
  std::vector<uint8_t>& cflags = bt.cflags;
  if (cl) {
    // values read in full (right operands, GEMV x), loop-carried ones included
    const auto& vo = q.r.ops;
    std::vector<char> full(q.r.is_vec.size(), 0);
    for (const BOp& o : vo)
      if (o.kind == OP_GEMM || o.kind == OP_GEMV) full[o.b] = 1;
    for (auto pr : {std::make_pair(q.G, q.gn), std::make_pair(q.F, q.fn),
                    std::make_pair(q.T, q.tn)})
      if (full[pr.first]) full[pr.second] = 1;
    std::vector<bool> bcast(vo.size());
    for (size_t k = 0; k < vo.size(); ++k) bcast[k] = vo[k].kind != OP_LOAD && full[vo[k].dst];
    cflags = cluster_flags(ops, bcast);
  }
  // device encoding: modes decided here, constants in a side table
  std::vector<DOp>& dev_ops = bt.dev_ops;
  dev_ops.resize(ops.size());
  std::vector<double>& csts = bt.csts;
  csts = {0.0};  // slot 0: unused default
  for (size_t k = 0; k < ops.size(); ++k) {
    const BOp& o = ops[k];
    DOp& d = dev_ops[k];
    d = DOp{};
    d.kind = (uint8_t)o.kind;
    d.sync = cl ? cflags[k] : (uint8_t)o.pad_;
    d.nterms = (uint8_t)o.nterms;
    d.dst = o.dst;
    d.a = o.a;
    d.b = o.b;
    d.c = o.c;
    for (int j = 0; j < kMaxLinTerms; ++j) d.t[j] = o.t[j];
    d.cidx = (int16_t)csts.size();
    d.prebar = (int16_t)(o.kind == OP_GEMM && (o.dst == o.a || o.dst == o.b));
    if (o.kind == OP_GEMM) {
      const bool hc = o.c >= 0;
      d.mode = (!hc && o.alpha == 1.0 && o.diag == 0.0)                     ? 0
               : (!hc && o.alpha == -1.0 && o.diag == 1.0)                  ? 1
               : (hc && o.alpha == 1.0 && o.beta == 1.0 && o.diag == 0.0)   ? 2
                                                                             : 3;
      csts.insert(csts.end(), {o.alpha, o.beta, o.diag});
    } else if (o.kind == OP_GEMV) {
      const bool hc = o.c >= 0;
      d.mode = (hc && o.alpha == 1.0 && o.beta == -1.0)    ? 1
               : (hc && o.alpha == -1.0 && o.beta == 1.0)  ? 2
                                                            : 3;
      csts.insert(csts.end(), {o.alpha, o.beta});
    } else if (o.kind == OP_LIN) {
      d.mode = (uint8_t)o.vec;
      csts.push_back(o.diag);
      for (int j = 0; j < o.nterms; ++j) csts.push_back(o.coef[j]);
    } else {
      d.mode = (uint8_t)o.vec;  // OP_LOAD: which matrix
    }
  }
  const size_t smem = (size_t)al.nmat * Gm::SLOT * sizeof(double) +
                      (size_t)al.nvec * NP * sizeof(double) + dev_ops.size() * sizeof(DOp) +
                      csts.size() * sizeof(double);
  if (smem > 227 * 1024) throw Error(kEInval, "resident program needs too much shared memory");
  bt.smem = smem;
  const size_t op_bytes = dev_ops.size() * sizeof(DOp);
  bt.blob.assign(op_bytes + csts.size() * sizeof(double), '\0');
  std::memcpy(&bt.blob[0], dev_ops.data(), op_bytes);
  std::memcpy(&bt.blob[op_bytes], csts.data(), csts.size() * sizeof(double));
  return bt;
}

template <int NP>
Counters launch(Ctx& c, Recipe& q, int64_t batch, int64_t n, const double* a, const double* b,
                const double* precond, const double* residual, int iters, const double* p_in,
                const double* f_in, const double* theta_in, double* p_io, double* f_io,
                double* theta_io, const ChunkGate* gate = nullptr) {
  using Gm = Geo<NP>;
  Counters per;
  for (const BOp& o : q.r.ops) {
    if (o.kind == OP_GEMM) per.mmm += 1;
    if (o.kind == OP_GEMV) per.mvm += 1;
  }
  per.mmm *= iters;
  per.mvm *= iters;
  if (batch == 0) return per;
  if (iters == 0) {  // outputs = inputs
    const size_t mat = (size_t)batch * n * n * sizeof(double), vec = (size_t)batch * n * 8;
    if (p_io != p_in) check(cudaMemcpyAsync(p_io, p_in, mat, cudaMemcpyDeviceToDevice, c.s), "copy");
    if (f_io != f_in) check(cudaMemcpyAsync(f_io, f_in, mat, cudaMemcpyDeviceToDevice, c.s), "copy");
    if (theta_io != theta_in)
      check(cudaMemcpyAsync(theta_io, theta_in, vec, cudaMemcpyDeviceToDevice, c.s), "copy");
    return per;
  }
  Built bt = build_program<NP>(q, batch, gate);
  const std::vector<BOp>& ops = bt.ops;
  const std::vector<DOp>& dev_ops = bt.dev_ops;
  const std::vector<double>& csts = bt.csts;
  const Alloc& al = bt.al;
  const int cl = bt.cl;
  const std::vector<uint8_t>& cflags = bt.cflags;
  const size_t smem = bt.smem;
  // program + constants, uploaded once per distinct program (handle cache)
  const size_t op_bytes = dev_ops.size() * sizeof(DOp);
  const std::string& blob = bt.blob;
  void* prog_dev = nullptr;
  {
    auto it = c.h->programs.find(blob);
    if (it != c.h->programs.end()) {
      prog_dev = it->second;
    } else {
      check(cudaMalloc(&prog_dev, blob.size()), "cudaMalloc");
      const cudaError_t err =
          cudaMemcpyAsync(prog_dev, blob.data(), blob.size(), cudaMemcpyHostToDevice, c.s);
      if (err == cudaSuccess) check(cudaStreamSynchronize(c.s), "sync");  // blob is freed below
      if (err != cudaSuccess) cudaFree(prog_dev);
      check(err, "memcpy program");
      c.h->programs.emplace(blob, prog_dev);
    }
  }
  BatchArgs args{};
  args.a = a;
  args.b = b;
  args.precond = precond;
  args.residual = residual;
  args.p_in = p_in;
  args.f_in = f_in;
  args.theta_in = theta_in;
  args.p_io = p_io;
  args.f_io = f_io;
  args.theta_io = theta_io;
  args.ops = reinterpret_cast<const DOp*>(prog_dev);
  args.nops = (int)ops.size();
  args.cst = reinterpret_cast<const double*>(reinterpret_cast<char*>(prog_dev) + op_bytes);
  args.ncst = (int)csts.size();
  args.nmat = al.nmat;
  args.nvec = al.nvec;
  args.n = (int)n;
  args.iters = iters;
  args.batch = batch;
  args.has_load = 0;
  args.last_load = -1;
  for (size_t k = 0; k < ops.size(); ++k)
    if (ops[k].kind == OP_LOAD) {
      args.has_load = 1;
      args.last_load = (int)k;
    }
  if (gate && gate->ready) {
    args.chunk_ready = gate->ready;
    args.chunk_done = gate->done;
    args.epoch = gate->epoch;
    args.chunk = gate->chunk;
  }
  args.sA = al.phys[q.A];
  args.sP = q.P >= 0 ? al.phys[q.P] : -1;
  args.sB = q.B >= 0 ? al.phys[q.B] : -1;
  args.sG = al.phys[q.G];
  args.sF = al.phys[q.F];
  args.sT = al.phys[q.T];
  args.sb = al.phys[q.bv];
  args.rG = al.phys[q.gn];
  args.rF = al.phys[q.fn];
  args.rT = al.phys[q.tn];
  if (cl) {
    auto kern = cl == 2 ? resident_cluster_kernel<2>
                : cl == 4 ? resident_cluster_kernel<4> : resident_cluster_kernel<8>;
#ifdef SI_HAVE_FIXED_C1
    // the program is byte for byte the baked config-1 one: straight-line kernel
    if (cl == 8 && !fixed_disabled() && std::getenv("SI_RESIDENT_PROF") == nullptr &&
        blob.size() == sizeof(FixedC1::blob) &&
        std::memcmp(blob.data(), FixedC1::blob, blob.size()) == 0)
      kern = resident_cluster_kernel<8, FixedC1>;
#endif
    check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
          "cudaFuncSetAttribute");
    long long* cprof = nullptr;
    const bool cwant = std::getenv("SI_RESIDENT_PROF") != nullptr;
    if (cwant) {
      check(cudaMalloc(&cprof, sizeof(long long) * (kMaxOps + 1)), "cudaMalloc");
      check(cudaMemset(cprof, 0, sizeof(long long) * (kMaxOps + 1)), "cudaMemset");
    }
    args.prof = cprof;
    const int64_t clusters = std::min<int64_t>(batch, std::max(1, num_sms_b() / cl));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(clusters * cl));
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check(cudaLaunchKernelEx(&cfg, kern, args), "resident cluster kernel launch");
    if (cwant) {
      std::vector<long long> hp(kMaxOps + 1);
      check(cudaMemcpy(hp.data(), cprof, sizeof(long long) * (kMaxOps + 1), cudaMemcpyDeviceToHost),
            "memcpy");
      cudaFree(cprof);
      const char* names[] = {"gemm", "gemv", "lin", "load"};
      std::fprintf(stderr, "[resident cluster %d] CTA0 cycles per op:\n", cl);
      for (size_t k = 0; k < ops.size(); ++k)
        std::fprintf(stderr, "  op %2zu %-4s dst %d a %d b %d c %d flags %d: %lld\n", k,
                     names[ops[k].kind], ops[k].dst, ops[k].a, ops[k].b, ops[k].c,
                     (int)cflags[k], hp[k]);
    }
    c.h->launches += 1;
    return per;
  }
  check(cudaFuncSetAttribute(resident_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem),
        "cudaFuncSetAttribute");
  int per_sm = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, resident_kernel<NP>,
                                                      Gm::THREADS, smem),
        "occupancy");
  if (per_sm < 1) throw Error(kEInval, "resident kernel does not fit on an SM");
  const int64_t grid = std::min<int64_t>(batch, (int64_t)num_sms_b() * per_sm);
  long long* prof = nullptr;
  const bool want_prof = std::getenv("SI_RESIDENT_PROF") != nullptr;
  if (want_prof) {
    check(cudaMalloc(&prof, sizeof(long long) * (kMaxOps + 1)), "cudaMalloc");
    check(cudaMemset(prof, 0, sizeof(long long) * (kMaxOps + 1)), "cudaMemset");
  }
  args.prof = prof;
  MV counter;  // dynamic system claims (released stream-ordered after the launch)
  if (batch > grid) {
    counter = alloc(c, 1, 1);
    check(cudaMemsetAsync(counter.v.p, 0, sizeof(unsigned long long), c.s), "memset");
    args.sys_counter = reinterpret_cast<unsigned long long*>(counter.v.p);
  }
  bool fixed = false;
#ifdef SI_HAVE_FIXED_C2
  // the launcher's program is byte for byte the baked one: straight-line kernel
  if constexpr (NP == 32) {
    if (!want_prof && !fixed_disabled() &&
        blob.size() == sizeof(FixedC2::blob) &&
        std::memcmp(blob.data(), FixedC2::blob, blob.size()) == 0) {
      check(cudaFuncSetAttribute(resident_kernel<NP, FixedC2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "cudaFuncSetAttribute");
      resident_kernel<NP, FixedC2><<<(unsigned)grid, Gm::THREADS, smem, c.s>>>(args);
      fixed = true;
    }
  }
#endif
  if (!fixed) resident_kernel<NP><<<(unsigned)grid, Gm::THREADS, smem, c.s>>>(args);
  if (want_prof) {
    std::vector<long long> h(kMaxOps + 1);
    check(cudaMemcpy(h.data(), prof, sizeof(long long) * (kMaxOps + 1), cudaMemcpyDeviceToHost),
          "memcpy");
    cudaFree(prof);
    const char* names[] = {"gemm", "gemv", "lin", "load"};
    long long tot = 0;
    for (size_t k = 0; k < ops.size(); ++k) tot += (k == 0 ? 0 : h[k]);
    std::fprintf(stderr, "[resident] CTA0 cycles per op (grid %lld, %d CTAs/SM, smem %zu B):\n",
                 (long long)grid, per_sm, smem);
    for (size_t k = 0; k < ops.size(); ++k)
      std::fprintf(stderr, "  op %2zu %-4s dst %d a %d b %d c %d: %lld\n", k, names[ops[k].kind],
                   ops[k].dst, ops[k].a, ops[k].b, ops[k].c, h[k]);
    std::fprintf(stderr, "  total (ops 1..) %lld\n", tot);
  }
  check(cudaGetLastError(), "resident kernel launch");
  c.h->launches += 1;
  return per;
}

}  // namespace

namespace {

Recipe composite_recipe(const std::vector<int>& rates, const std::vector<const PlanNode*>& plans,
                        int order_n) {
  Recipe q = new_recipe();
  record_plain(q);
  // composite_step (newton_schulz.py:177-228).  The NS part S_n(F) G is
  // evaluated first (the parts are independent of it) so G and F die early;
  // S^-1 and B are streamed in for the parts and die after the last one.
  const int nsp = q.r.horner(q.F, q.G, order_n);
  // S^-1 and B: resident for the whole run (pinned slots), or streamed in every
  // iteration through registers (OP_LOAD) when their two slots would cost a
  // CTA per SM (SI_RESIDENT_PIN_SPLIT=0/1 overrides)
  bool pin = false;
  if (const char* env = std::getenv("SI_RESIDENT_PIN_SPLIT")) pin = std::atoi(env) != 0;
  int P, B;
  if (pin) {
    q.P = P = q.r.fresh(false);
    q.B = B = q.r.fresh(false);
  } else {
    P = q.r.load(0);
    B = q.r.load(1);
  }
  std::vector<int> ts, gs;
  for (size_t i = 0; i < rates.size(); ++i) {
    const int ti = q.r.geometric(B, P, rates[i], q.A, plans[i]);
    ts.push_back(ti);
    gs.push_back(q.r.residual(ti, q.A));
  }
  int tc = ts[0], rc = gs[0];
  for (size_t i = 1; i < ts.size(); ++i) {
    tc = q.r.gemm(rc, ts[i], 1.0, tc, 1.0);
    rc = q.r.gemm(rc, gs[i]);
  }
  q.gn = q.r.gemm(rc, nsp, 1.0, tc, 1.0);
  q.fn = q.r.residual(q.gn, q.A);
  defer_theta_update(q);
  return q;
}

}  // namespace

namespace {
std::string program_source(const Built& bt) {
  std::string out;
  char buf[256];
  std::snprintf(buf, sizeof(buf),
                "  static constexpr bool kFixed = true;\n  static constexpr int nops = %zu;\n"
                "  static constexpr DOp ops[%zu] = {\n",
                bt.dev_ops.size(), bt.dev_ops.size());
  out += buf;
  for (const DOp& d : bt.dev_ops) {
    std::snprintf(buf, sizeof(buf),
                  "      {%d, %d, %d, %d, %d, %d, %d, %d, {%d, %d, %d, %d, %d, %d}, %d, %d, {0, 0}},\n",
                  d.kind, d.mode, d.sync, d.nterms, d.dst, d.a, d.b, d.c, d.t[0], d.t[1], d.t[2],
                  d.t[3], d.t[4], d.t[5], d.cidx, d.prebar);
    out += buf;
  }
  out += "  };\n";
  std::snprintf(buf, sizeof(buf), "  static constexpr unsigned char blob[%zu] = {", bt.blob.size());
  out += buf;
  for (size_t i = 0; i < bt.blob.size(); ++i) {
    std::snprintf(buf, sizeof(buf), "%s%s%u", i ? "," : "", i % 24 == 0 ? "\n      " : "",
                  (unsigned)(unsigned char)bt.blob[i]);
    out += buf;
  }
  out += "};\n";
  return out;
}
}  // namespace

std::string resident_program_source(int64_t n, const std::vector<int>& rates,
                                    const std::vector<const PlanNode*>& plans, int order_n) {
  if (n > 32) throw Error(kEInval, "the baked program is for n <= 32");
  Recipe q = composite_recipe(rates, plans, order_n);
  Built bt = build_program<32>(q, int64_t(1) << 30, nullptr);
  return program_source(bt);
}

Counters batched_composite_richardson(Ctx& c, int64_t batch, int64_t n, const double* a,
                                      const double* b, const double* precond,
                                      const double* residual, const std::vector<int>& rates,
                                      const std::vector<const PlanNode*>& plans, int order_n,
                                      int iters, const double* p_in, const double* f_in,
                                      const double* theta_in, double* p_io, double* f_io,
                                      double* theta_io, const ChunkGate* gate) {
  Recipe q = composite_recipe(rates, plans, order_n);
  if (n <= 32)
    return launch<32>(c, q, batch, n, a, b, precond, residual, iters, p_in, f_in, theta_in, p_io,
                      f_io, theta_io, gate);
  return launch<64>(c, q, batch, n, a, b, precond, residual, iters, p_in, f_in, theta_in, p_io,
                    f_io, theta_io, gate);
}

namespace {
Recipe ns_recipe(int order, const PlanNode* plan) {
  Recipe q = new_recipe();
  record_plain(q);
  // ns_step (newton_schulz.py:150-174)
  const int gnew = plan ? q.r.eval(*plan, q.F, q.G, q.A) : q.r.horner(q.F, q.G, order);
  q.gn = gnew == q.G ? q.r.copy(q.G) : gnew;
  q.fn = q.r.residual(q.gn, q.A);
  // (no defer_theta_update here: in the cluster kernel the deferred GEMV
  // reads G, whose slot the next product overwrites in place -- a barrier
  // either way -- and the config-1 iteration measured slower)
  return q;
}
}  // namespace

std::string resident_program_source_ns(int64_t n, int order, int cl) {
  if (n <= 32 || n > 64) throw Error(kEInval, "the baked cluster program is for 32 < n <= 64");
  Recipe q = ns_recipe(order, nullptr);
  Built bt = build_program<64>(q, 1, nullptr, cl);
  return program_source(bt);
}

Counters batched_ns_richardson(Ctx& c, int64_t batch, int64_t n, const double* a, const double* b,
                               int order, const PlanNode* plan, int iters, const double* p_in,
                               const double* f_in, const double* theta_in, double* p_io,
                               double* f_io, double* theta_io) {
  Recipe q = ns_recipe(order, plan);
  if (n <= 32)
    return launch<32>(c, q, batch, n, a, b, nullptr, nullptr, iters, p_in, f_in, theta_in, p_io,
                      f_io, theta_io);
  return launch<64>(c, q, batch, n, a, b, nullptr, nullptr, iters, p_in, f_in, theta_in, p_io,
                    f_io, theta_io);
}

}  // namespace si
