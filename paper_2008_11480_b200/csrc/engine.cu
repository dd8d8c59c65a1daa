// Native step engine.  Every function cites the reference code it mirrors; the
// GEMM DAG (which products, in which order, with which element-wise op after
// each) is the reference's, so the mmm/mvm counters match matrix_core.py:71-98
// tick for tick, while the element-wise ops are fused into the GEMM epilogues.
#include "engine.hpp"
#include "ozaki.hpp"
#include "shard.hpp"

#include <algorithm>
#include <cstring>

namespace si {

thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* get_error() { return g_err.c_str(); }

void check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation)
    throw Error(kENoMem, std::string(what) + ": " + cudaGetErrorString(e));
  throw Error(kECuda, std::string(what) + ": " + cudaGetErrorString(e));
}

Buf::~Buf() {
  if (!p) return;
  if (external)
    h->free_fn(h->alloc_ctx, p, free_stream);
  else
    cudaFreeAsync(p, free_stream);
}

MV view(double* p, int64_t rows, int64_t cols, int64_t ld) {
  MV m;
  m.v.p = p;
  m.v.rows = rows;
  m.v.cols = cols;
  m.v.ld = ld;
  return m;
}

MV alloc(Ctx& c, int64_t rows, int64_t cols) {
  auto b = std::make_shared<Buf>();
  b->free_stream = c.root;
  b->h = c.h;
  void* p = nullptr;
  const size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(rows * cols, 1);
  if (c.h->alloc_fn) {
    // external allocator, always associated with the root stream
    p = c.h->alloc_fn(c.h->alloc_ctx, bytes, c.root);
    if (!p) throw Error(kENoMem, "external allocator returned NULL");
    b->external = true;
    if (c.s != c.root) {
      // a branch stream uses memory handed out in root-stream order
      cudaEvent_t e;
      check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      check(cudaEventRecord(e, c.root), "cudaEventRecord");
      check(cudaStreamWaitEvent(c.s, e, 0), "cudaStreamWaitEvent");
      cudaEventDestroy(e);
    }
  } else {
    check(cudaMallocFromPoolAsync(&p, bytes, c.h->pool, c.s), "cudaMallocFromPoolAsync");
  }
  b->p = static_cast<double*>(p);
  if (c.keep) c.keep->push_back(b);
  MV m = view(b->p, rows, cols, cols);
  m.own = b;
  return m;
}

// ---------------------------------------------------------------------------
// products
// ---------------------------------------------------------------------------

void Ctx::await_ptr(const void* p) {
  for (Await& a : awaits)
    if (!a.done && a.base == p) {
      check(cudaStreamWaitEvent(s, a.ev, 0), "cudaStreamWaitEvent");
      a.done = true;
    }
}

const PanelWait* Ctx::gate_of(const void* p) const {
  for (const Gate& g : gates)
    if (g.base == p && !g.stream_done) return &g.pw;
  return nullptr;
}

void Ctx::gate_stream(const void* p) {
  for (Gate& g : gates)
    if (g.base == p && !g.stream_done) {
      for (int i = 0; i < g.pw.npanels; ++i)
        check(stream_wait_u32(g.pw.ready + i, g.pw.epoch, s), "panel wait");
      g.stream_done = true;
    }
}

struct Ctx::OzSide {
  const void* ptr;
  int64_t rows, cols, ld, k;
  int nmod;
  bool b_side;
  MV buf;
  oz::Side side;
};

void keep_stable(Ctx& c, const MV& v) {
  if (c.s != c.root || !v.v.p) return;
  const size_t bytes = sizeof(double) * (size_t)(v.v.rows > 0 ? (v.v.rows - 1) * v.v.ld + v.v.cols : 0);
  c.stable.push_back({reinterpret_cast<const char*>(v.v.p), bytes});
  c.stable_keep.push_back(v);
}

namespace {
constexpr size_t kOzSideMaxBytes = (size_t)8 << 30;  // keep sides up to n = 16384 x 16384

// The kept scales + planes of operand `m` (A side: rows of A; B side: columns
// of B) of an emulated product with inner dimension k, or nullptr when `m` is
// not a stable input of this call (or its side does not fit the budget).
oz::Side* oz_side(Ctx& c, const Mat& m, bool b_side, int64_t k, int nmod) {
  if (c.s != c.root || c.stable.empty() || m.rows <= 0) return nullptr;
  // the whole matrix (rows x cols at ld) inside one stable range
  const char* lo = reinterpret_cast<const char*>(m.p);
  const char* hi = lo + sizeof(double) * (size_t)((m.rows - 1) * m.ld + m.cols);
  bool inside = false;
  for (const auto& r : c.stable)
    if (lo >= r.base && hi <= r.base + r.bytes) inside = true;
  if (!inside) return nullptr;
  for (auto& e : c.oz_sides)
    if (e->ptr == m.p && e->rows == m.rows && e->cols == m.cols && e->ld == m.ld && e->k == k &&
        e->nmod == nmod && e->b_side == b_side)
      return &e->side;
  const int64_t n = b_side ? m.cols : m.rows;
  const size_t bytes = oz::side_bytes(n, k, nmod);
  if (bytes > kOzSideMaxBytes) return nullptr;
  auto e = std::make_shared<Ctx::OzSide>();
  try {
    e->buf = alloc(c, 1, (int64_t)((bytes + 7) / 8));
  } catch (const Error& ex) {
    if (ex.code == kENoMem) return nullptr;  // no room: compute per product
    throw;
  }
  e->ptr = m.p;
  e->rows = m.rows;
  e->cols = m.cols;
  e->ld = m.ld;
  e->k = k;
  e->nmod = nmod;
  e->b_side = b_side;
  auto* base = reinterpret_cast<uint8_t*>(e->buf.v.p);
  e->side.scale = reinterpret_cast<unsigned long long*>(base);
  e->side.planes = reinterpret_cast<int8_t*>(base + ((n * 8 + 255) & ~(int64_t)255));
  e->side.ready = false;
  c.oz_sides.push_back(e);
  return &e->side;
}
}  // namespace

// fused-norm slots of one product (Ctx::sq): a fresh slot buffer, appended
static double* sq_slots_for(Ctx& c, int64_t slots) {
  MV part = alloc(c, 1, slots);
  c.sq->parts.emplace_back(part, slots);
  return part.v.p;
}

// products without a fused epilogue partial (GEMV, small-n generic kernel):
// one partial pass over the stored values
static cudaError_t unfused_sq(Ctx& c, const Mat& d) {
  double* part = sq_slots_for(c, sumsq_partials());
  c.h->launches += 1;
  return launch_sumsq_partials(d, part, c.s);
}

void finish_sq(Ctx& c, const Ctx::SqAcc& acc, const Mat& F, double* out) {
  if (acc.parts.empty()) {
    MV work = alloc(c, 1, (int64_t)reduce_work_elems(F));
    check(launch_sumsq(F, out, work.v.p, c.s), "sumsq");
    c.h->launches += 2;
    return;
  }
  for (size_t i = 0; i < acc.parts.size(); ++i) {
    check(launch_sum_slots(acc.parts[i].first.v.p, acc.parts[i].second, out, i > 0, c.s),
          "sum slots");
    c.h->launches += 1;
  }
}

void gemm(Ctx& c, const MV& D, const MV& A, const MV& B, double alpha, const MV* C, double beta,
          double diag, bool mv, int64_t doff, const PanelWait* pw) {
  if (c.shard) {
    // block-row sharded: this rank's rows of A @ B (+ C rows, diag at the
    // block's global diagonal), B gathered if it is sharded; a replicated
    // output is completed by an all-gather of its row blocks
    Shard* sh = c.shard;
    const MV a = shard_rows(c, A), b = shard_full(c, B);
    MV cr;
    if (C) cr = shard_rows(c, *C);
    const MV d = shard_rows(c, D);
    c.shard = nullptr;
    try {
      gemm(c, d, a, b, alpha, C ? &cr : nullptr, beta, diag, mv, doff + sh->r0, pw);
    } catch (...) {
      c.shard = sh;
      throw;
    }
    c.shard = sh;
    if (!D.local) shard_gather_into(c, D);
    return;
  }
  if (A.v.cols != B.v.rows || D.v.rows != A.v.rows || D.v.cols != B.v.cols)
    throw Error(kEInval, "dimension mismatch in product");
  if (C && (C->v.rows != D.v.rows || C->v.cols != D.v.cols))
    throw Error(kEInval, "dimension mismatch in epilogue operand");
  Epilogue e;
  e.alpha = alpha;
  e.beta = C ? beta : 0.0;
  e.diag = diag;
  e.doff = doff;
  e.c = C ? C->v.p : nullptr;
  e.ldc = C ? C->v.ld : 0;
  Mat d = D.v;
  cudaError_t err;
  Handle* h = c.h;
  const bool collect_sq = c.sq && d.p >= c.sq_lo && d.p < c.sq_hi && d.rows > 0 && d.cols > 0;
  if (!c.awaits.empty()) {
    c.await_ptr(A.v.p);
    c.await_ptr(B.v.p);
    if (C) c.await_ptr(C->v.p);
  }
  const bool use_tma = d.rows > 0 && d.cols > 4 && std::max(d.rows, d.cols) >= 128 &&
                       A.v.cols > 0 && tma_eligible(A.v, B.v, d, e);
  // Ozaki-II products (backend 1): inputs still in flight are awaited on the
  // stream (whole operands); the residue kernels have no in-kernel gates
  const bool use_oz = h->gemm_backend == 1 && d.rows >= h->oz_min_dim &&
                      d.cols >= h->oz_min_dim && A.v.cols >= h->oz_min_dim &&
                      A.v.cols <= oz::kMaxK;
  const bool in_kernel_gates = use_tma && !use_oz;
  // inputs still arriving in row panels: in-kernel gates for A rows / B k-slabs
  // of the DMMA GEMM, stream waits for everything else
  const PanelWait* pwa = nullptr;
  const PanelWait* oz_rows = nullptr;  // emulated product: rows of A waited per row chunk
  if (!c.gates.empty()) {
    if (in_kernel_gates) {
      pwa = c.gate_of(A.v.p);
      if (!pw) pw = c.gate_of(B.v.p);
      if (C && C->v.p != B.v.p) c.gate_stream(C->v.p);  // C == B: its panels gate the k-loop
    } else {
      // (only for panels of >= 2048 rows: smaller row chunks cost more in
      // partial INT8 waves than the copy they hide)
      if (use_oz && A.v.p != B.v.p && (!C || C->v.p != A.v.p) && A.v.rows == d.rows) {
        oz_rows = c.gate_of(A.v.p);
        for (int p = 0; oz_rows && p < oz_rows->npanels; ++p)
          if (oz_rows->bounds[p + 1] - oz_rows->bounds[p] < 2048) oz_rows = nullptr;
      }
      if (!oz_rows) c.gate_stream(A.v.p);
      c.gate_stream(B.v.p);
      if (C) c.gate_stream(C->v.p);
    }
  }
  const bool gated = pw && pw->ready && pw->npanels > 0;
  if (gated && !in_kernel_gates) {
    // kernels without the in-kernel gate: the stream waits for every panel
    for (int p = 0; p < pw->npanels; ++p)
      check(stream_wait_u32(pw->ready + p, pw->epoch, c.s), "panel wait");
  }
  if (d.rows == 0 || d.cols == 0) {
    err = cudaSuccess;
  } else if (use_oz) {
    Handle::ProfRec rec{};
    auto draw = [&](cudaEvent_t* ev) {
      if (h->prof_pool.empty()) {
        check(cudaEventCreate(ev), "cudaEventCreate");
      } else {
        *ev = h->prof_pool.back();
        h->prof_pool.pop_back();
      }
    };
    if (h->profiling) {
      for (cudaEvent_t* ev : {&rec.start, &rec.stop}) draw(ev);
      rec.flops = 2.0 * (double)d.rows * (double)d.cols * (double)A.v.cols;
      check(cudaEventRecord(rec.start, c.s), "cudaEventRecord");
    }
    // workspace: the configured chunking first; when the allocator cannot
    // serve it, smaller row x column chunks (halved each retry; the B-side
    // planes are then rebuilt per row chunk)
    oz::Work w;
    w.max_cols = h->oz_max_cols;
    w.max_rows = h->oz_max_rows;
    w.variant = h->oz_variant;
    oz::RowHook row_hook;
    if (oz_rows) {
      // A's rows still arriving in panels: one row chunk per panel, each
      // waiting for its own panels only, so the product runs behind the copy
      const PanelWait gate = *oz_rows;
      int64_t prow = d.rows;
      for (int p = 0; p < gate.npanels; ++p)
        prow = std::min<int64_t>(prow, gate.bounds[p + 1] - gate.bounds[p]);
      w.max_rows = w.max_rows > 0 ? std::min(w.max_rows, prow) : prow;
      row_hook = [&c, gate](int64_t r0, int64_t r1) {
        for (int p = 0; p < gate.npanels; ++p)
          if (gate.bounds[p] < r1 && gate.bounds[p + 1] > r0)
            check(stream_wait_u32(gate.ready + p, gate.epoch, c.s), "panel wait");
      };
    }
    // A branch context keeps every buffer it allocates until its join, so its
    // products share one workspace (stream-ordered on the branch stream); on
    // the root stream each product's workspace is released right after it.
    const bool reuse_ws = c.s != c.root;
    MV ws;
    for (int level = 0;; ++level) {
      w.bytes = oz::workspace_bytes(d.rows, d.cols, A.v.cols, h->oz_nmod, w.max_cols, w.max_rows);
      if (reuse_ws && c.oz_ws.own && c.oz_ws_bytes >= w.bytes) {
        ws = c.oz_ws;
        break;
      }
      try {
        ws = alloc(c, 1, (int64_t)((w.bytes + 7) / 8));
        if (reuse_ws) {
          c.oz_ws = ws;
          c.oz_ws_bytes = w.bytes;
        }
        break;
      } catch (const Error& ex) {
        if (ex.code != kENoMem || level == 4 || (w.max_rows > 0 && w.max_rows <= 1024)) throw;
        const int64_t rows = w.max_rows > 0 ? w.max_rows : d.rows;
        const int64_t cols = w.max_cols > 0 ? std::min(w.max_cols, d.cols) : d.cols;
        w.max_rows = std::max<int64_t>(1024, rows / 2);
        w.max_cols = std::max<int64_t>(1024, cols / 2);
      }
    }
    w.base = reinterpret_cast<uint8_t*>(ws.v.p);
    int64_t nl = 0;
    // one event pair per INT8 tensor-core launch (column chunks)
    Handle::ProfRec rec8{};
    oz::I8Hook hook;
    if (h->profiling) {
      hook = [&](bool begin, double ops) {
        if (begin) {
          rec8 = Handle::ProfRec{};
          draw(&rec8.start);
          draw(&rec8.stop);
          rec8.flops = ops;
          check(cudaEventRecord(rec8.start, c.s), "cudaEventRecord");
        } else {
          check(cudaEventRecord(rec8.stop, c.s), "cudaEventRecord");
          h->prof_i8.push_back(rec8);
        }
      };
    }
    oz::Side* as = oz_side(c, A.v, false, A.v.cols, h->oz_nmod);
    oz::Side* bs = oz_side(c, B.v, true, A.v.cols, h->oz_nmod);
    if (collect_sq) e.sq = sq_slots_for(c, oz::sq_slots(d.rows, d.cols, A.v.cols, h->oz_nmod, w));
    err = oz::launch_gemm(A.v, B.v, d, e, h->oz_nmod, w, c.s, &nl, hook, as, bs, row_hook);
    if (oz_rows) c.gate_stream(A.v.p);  // every panel waited (no-ops by now): later readers
    h->launches += nl;
    if (h->profiling && err == cudaSuccess) {
      check(cudaEventRecord(rec.stop, c.s), "cudaEventRecord");
      h->prof.push_back(rec);
    }
  } else if (d.cols <= 4) {
    err = launch_gemv(A.v, B.v, d, e, c.s);
    h->launches += 1;
    if (collect_sq && err == cudaSuccess) err = unfused_sq(c, d);
  } else if (use_tma) {
    if (collect_sq) e.sq = sq_slots_for(c, gemm_tma_sq_slots(d.rows, d.cols));
    Handle::ProfRec rec{};
    if (h->profiling) {
      for (cudaEvent_t* ev : {&rec.start, &rec.stop}) {
        if (h->prof_pool.empty()) {
          check(cudaEventCreate(ev), "cudaEventCreate");
        } else {
          *ev = h->prof_pool.back();
          h->prof_pool.pop_back();
        }
      }
      rec.flops = 2.0 * (double)d.rows * (double)d.cols * (double)A.v.cols;
      check(cudaEventRecord(rec.start, c.s), "cudaEventRecord");
    }
    err = launch_gemm_tma(A.v, B.v, d, e, c.s, gated ? pw : nullptr, pwa);
    h->launches += 1;
    if (h->profiling && err == cudaSuccess) {
      check(cudaEventRecord(rec.stop, c.s), "cudaEventRecord");
      h->prof.push_back(rec);
    }
  } else {
    err = launch_gemm_generic(A.v, B.v, d, e, c.s);
    h->launches += 1;
    if (collect_sq && err == cudaSuccess) err = unfused_sq(c, d);
  }
  check(err, "gemm launch");
  if (mv)
    c.ctr.mvm += 1;
  else
    c.ctr.mmm += 1;
}

MV alloc_like(Ctx& c, const MV& x) {
  if (!c.shard) return alloc(c, x.v.rows, x.v.cols);
  MV d = alloc(c, c.shard->r1 - c.shard->r0, x.v.cols);
  d.local = true;
  return d;
}

MV identity_like(Ctx& c, const MV& x, double scale) {
  MV d = alloc_like(c, x);
  if (c.shard) {  // this rank's rows of scale * I
    check(launch_lincomb(d.v, scale, c.shard->r0, 0, nullptr, nullptr, c.s), "identity rows");
  } else {
    check(launch_fill_identity(d.v, scale, c.s), "identity");
  }
  c.h->launches += 1;
  return d;
}

MV gemm_new(Ctx& c, const MV& A, const MV& B, double alpha, const MV* C, double beta, double diag,
            bool mv) {
  MV D;
  if (c.shard) {  // this rank's rows of the product
    D = alloc(c, c.shard->r1 - c.shard->r0, B.v.cols);
    D.local = true;
  } else {
    D = alloc(c, A.v.rows, B.v.cols);
  }
  gemm(c, D, A, B, alpha, C, beta, diag, mv);
  return D;
}

// identity(n) - mat_mul(X, A)  (the residual form)
MV residual(Ctx& c, const MV& X, const MV& A) { return gemm_new(c, X, A, -1.0, nullptr, 0.0, 1.0); }
void residual_into(Ctx& c, const MV& D, const MV& X, const MV& A) {
  gemm(c, D, X, A, -1.0, nullptr, 0.0, 1.0);
}

void copy_into(Ctx& c, const MV& D, const MV& X) {
  if (c.shard) {
    const MV d = shard_rows(c, D), x = shard_rows(c, X);
    Shard* sh = c.shard;
    c.shard = nullptr;
    copy_into(c, d, x);
    c.shard = sh;
    if (!D.local) shard_gather_into(c, D);
    return;
  }
  if (D.v.p == X.v.p) return;
  if (!c.awaits.empty()) c.await_ptr(X.v.p);
  if (!c.gates.empty()) c.gate_stream(X.v.p);
  Mat d = D.v;
  check(launch_copy(d, X.v, c.s), "copy");
  c.h->launches += 1;
}

MV lincomb(Ctx& c, double cdiag, const std::vector<std::pair<double, const MV*>>& terms,
           int64_t rows, int64_t cols) {
  int64_t doff = 0;
  std::vector<MV> loc;
  if (c.shard) {  // this rank's rows of every term; cdiag * I on the block's diagonal
    rows = c.shard->r1 - c.shard->r0;
    doff = c.shard->r0;
    for (auto& t : terms) loc.push_back(shard_rows(c, *t.second));
  }
  MV D = alloc(c, rows, cols);
  D.local = c.shard != nullptr;
  if ((int)terms.size() > kMaxLinTerms) throw Error(kEInval, "too many lin terms");
  double coef[kMaxLinTerms];
  Mat xs[kMaxLinTerms];
  for (size_t i = 0; i < terms.size(); ++i) {
    coef[i] = terms[i].first;
    xs[i] = c.shard ? loc[i].v : terms[i].second->v;
    if (!c.awaits.empty()) c.await_ptr(xs[i].p);
    if (!c.gates.empty()) c.gate_stream(xs[i].p);
  }
  check(launch_lincomb(D.v, cdiag, doff, (int)terms.size(), coef, xs, c.s), "lincomb");
  c.h->launches += 1;
  return D;
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------

namespace {
struct Decoder {
  const int32_t* code;
  int64_t len, pos = 0;
  const double* consts;
  int64_t nconsts;
  int32_t next() {
    if (pos >= len) throw Error(kEInval, "malformed plan: truncated");
    return code[pos++];
  }
  double cst(int32_t slot) {
    if (slot < 0 || slot >= nconsts) throw Error(kEInval, "malformed plan: const slot");
    return consts[slot];
  }
  PlanPtr node(int depth) {
    if (depth > 16) throw Error(kEInval, "malformed plan: too deep");
    auto n = std::make_shared<PlanNode>();
    n->kind = next();
    switch (n->kind) {
      case 0:
        n->h = next();
        if (n->h < 1) throw Error(kEInval, "Horner order must be >= 1");
        break;
      case 1:
        n->p = next();
        n->w = next();
        if (n->p < 0 || n->w < 1) throw Error(kEInval, "Split requires p >= 0 and w >= 1");
        if (next()) n->inner = node(depth + 1);
        if (next()) n->outer = node(depth + 1);
        if (n->p >= 1 && !n->inner) throw Error(kEInval, "Split with p >= 1 needs an inner node");
        if (n->w >= 2 && !n->outer) throw Error(kEInval, "Split with w >= 2 needs an outer node");
        break;
      case 2:
        n->inner = node(depth + 1);
        break;
      case 3: {
        n->order = next();
        n->nregs = next();
        const int ninstr = next();
        if (n->nregs < 2 || ninstr < 0) throw Error(kEInval, "malformed table form");
        for (int i = 0; i < ninstr; ++i) {
          Instr ins;
          ins.op = next();
          ins.dst = next();
          ins.a = ins.b = -1;
          ins.cconst = 0.0;
          if (ins.op == 0) {
            ins.a = next();
            ins.b = next();
          } else if (ins.op == 1) {
            ins.a = next();
          } else if (ins.op == 2) {
            ins.cconst = cst(next());
            const int nt = next();
            for (int t = 0; t < nt; ++t) {
              const double cf = cst(next());
              ins.terms.emplace_back(cf, next());
            }
          } else {
            throw Error(kEInval, "malformed table form: opcode");
          }
          auto okreg = [&](int r) { return r >= 0 && r < n->nregs; };
          if (!okreg(ins.dst) || (ins.op <= 1 && !okreg(ins.a)) || (ins.op == 0 && !okreg(ins.b)))
            throw Error(kEInval, "malformed table form: register");
          for (auto& t : ins.terms)
            if (!okreg(t.second)) throw Error(kEInval, "malformed table form: register");
          n->prog.push_back(std::move(ins));
        }
        break;
      }
      default:
        throw Error(kEInval, "malformed plan: node kind");
    }
    return n;
  }
};
}  // namespace

int plan_order_of(const PlanNode& n) {
  switch (n.kind) {
    case 0:
      return n.h;
    case 1: {
      if (n.p >= 1 && plan_order_of(*n.inner) != n.p + 1)
        throw Error(kEInval, "Split inner order != p + 1");
      if (n.w >= 2 && plan_order_of(*n.outer) != n.w) throw Error(kEInval, "Split outer order != w");
      return n.w * (n.p + 1);
    }
    case 2:
      return plan_order_of(*n.inner) + 1;
    default:
      return n.order;
  }
}

PlanPtr decode_plan(const int32_t* code, int64_t len, const double* consts, int64_t nconsts) {
  if (!code || len <= 0) throw Error(kEInval, "empty plan");
  Decoder d{code, len, 0, consts, nconsts};
  PlanPtr p = d.node(0);
  if (d.pos != len) throw Error(kEInval, "malformed plan: trailing data");
  plan_order_of(*p);
  return p;
}

// ---------------------------------------------------------------------------
// evaluators
// ---------------------------------------------------------------------------

// st:263-267  z <- y z + x, h-1 times (each product + add fused in one GEMM)
MV horner(Ctx& c, const MV& y, const MV& x, int h) {
  MV z = x;
  for (int i = 0; i < h - 1; ++i) z = gemm_new(c, y, z, 1.0, &x, 1.0);
  return z;
}

// st:326-356 with the supplied Y (form_y handled by the caller)
MV factored(Ctx& c, const MV& y, const MV& x, const MV& a, int p, int w) {
  MV u = (p == 0) ? x : horner(c, y, x, p + 1);
  if (w == 1) return u;
  MV q = (p == 0) ? y : residual(c, u, a);
  return horner(c, q, u, w);
}

// st:359-382  straight-line program; a Mul whose only use is the very next
// Lin "0*I + 1*X + 1*mul" is fused into that GEMM's epilogue (identical
// rounding: numpy computes fl(X + fl(Y@Z)), the epilogue fl(acc + X)).
static MV run_program(Ctx& c, const PlanNode& node, const MV& y, const MV& x, const MV& a) {
  const auto& prog = node.prog;
  const int nr = node.nregs;
  std::vector<MV> env(nr);
  std::vector<int> last_use(nr, -1);
  for (int i = 0; i < (int)prog.size(); ++i) {
    const Instr& in = prog[i];
    if (in.a >= 0) last_use[in.a] = i;
    if (in.b >= 0) last_use[in.b] = i;
    for (auto& t : in.terms) last_use[t.second] = i;
  }
  env[0] = y;
  env[1] = x;
  int result = prog.empty() ? 1 : prog.back().dst;
  auto need = [&](int r) -> const MV& {
    if (!env[r].v.p && env[r].v.rows == 0) throw Error(kEInval, "malformed table form: unset register");
    return env[r];
  };
  for (int i = 0; i < (int)prog.size(); ++i) {
    const Instr& in = prog[i];
    if (in.op == 0) {
      // fusion candidate: next is lin(dst2, 0, [(1, other), (1, in.dst)]) or reversed,
      // and in.dst is not used after it.
      bool fused = false;
      if (i + 1 < (int)prog.size()) {
        const Instr& nx = prog[i + 1];
        if (nx.op == 2 && nx.cconst == 0.0 && nx.terms.size() == 2 && nx.terms[0].first == 1.0 &&
            nx.terms[1].first == 1.0 && last_use[in.dst] == i + 1 && in.dst != nx.dst) {
          int other = -1;
          if (nx.terms[1].second == in.dst && nx.terms[0].second != in.dst) other = nx.terms[0].second;
          if (nx.terms[0].second == in.dst && nx.terms[1].second != in.dst) other = nx.terms[1].second;
          if (other >= 0) {
            env[nx.dst] = gemm_new(c, need(in.a), need(in.b), 1.0, &need(other), 1.0);
            ++i;
            fused = true;
          }
        }
      }
      if (!fused) env[in.dst] = gemm_new(c, need(in.a), need(in.b));
    } else if (in.op == 1) {
      env[in.dst] = residual(c, need(in.a), a);
    } else {
      std::vector<std::pair<double, const MV*>> terms;
      for (auto& t : in.terms) terms.emplace_back(t.first, &need(t.second));
      env[in.dst] = lincomb(c, in.cconst, terms, x.v.rows, x.v.cols);
    }
    // release dead temporaries (never Y/X or the result)
    for (int r = 2; r < nr; ++r)
      if (r != result && last_use[r] >= 0 && last_use[r] <= i && env[r].own) env[r] = MV{};
  }
  return env[result];
}

// st:385-405
MV eval_node(Ctx& c, const PlanNode& node, const MV& y, const MV& x, const MV& a) {
  switch (node.kind) {
    case 0:
      return horner(c, y, x, node.h);
    case 1: {
      MV u = (node.p == 0) ? x : eval_node(c, *node.inner, y, x, a);
      if (node.w == 1) return u;
      MV q = (node.p == 0) ? y : residual(c, u, a);
      return eval_node(c, *node.outer, q, u, a);
    }
    case 2: {
      MV z = eval_node(c, *node.inner, y, x, a);
      return gemm_new(c, y, z, 1.0, &x, 1.0);  // x + y z
    }
    default:
      return run_program(c, node, y, x, a);
  }
}

// mc:137-151
MV mat_pow_counted(Ctx& c, const MV& y, int e) {
  if (e == 0) return identity_like(c, y);
  MV base = y, result;
  bool have = false;
  while (e > 0) {
    if (e & 1) {
      result = have ? gemm_new(c, result, base) : base;
      have = true;
    }
    e >>= 1;
    if (e) base = gemm_new(c, base, base);
  }
  return result;
}

// st:432-457
MV geometric(Ctx& c, const MV& y, const MV& x, int order, const MV& a, const PlanNode* base) {
  if (order < 1) throw Error(kEInval, "order must be >= 1");
  if (order == 1) {
    MV d = alloc_like(c, x);
    copy_into(c, d, x);
    return d;
  }
  if (order <= 64) {
    if (!base || plan_order_of(*base) != order) throw Error(kEInval, "missing plan for geometric order");
    return eval_node(c, *base, y, x, a);
  }
  const int half = order / 2;
  MV t = geometric(c, y, x, half, a, base);
  MV yh = mat_pow_counted(c, y, half);
  MV z = gemm_new(c, yh, t, 1.0, &t, 1.0);  // t + y^half t
  if (order % 2) z = gemm_new(c, y, z, 1.0, &x, 1.0);
  return z;
}

// ---------------------------------------------------------------------------
// fork / join (executor hook: newton_schulz.py:275-285, richardson.py:556-566)
// ---------------------------------------------------------------------------

static cudaEvent_t get_event(Handle* h, size_t i) {
  while (h->events.size() <= i) {
    cudaEvent_t e;
    check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    h->events.push_back(e);
  }
  return h->events[i];
}

Fork::Fork(Ctx& c) : parent(c) {
  cudaEvent_t e = get_event(c.h, 0);
  check(cudaEventRecord(e, c.s), "cudaEventRecord");
  evs.push_back(e);
}

Ctx Fork::branch(int i) {
  if (i < 0 || i >= Handle::kSide) throw Error(kEInval, "too many branches");
  Ctx ch(parent.h, parent.root);
  ch.s = parent.h->side[i];
  ch.keep = std::make_shared<std::vector<std::shared_ptr<Buf>>>();
  ch.awaits = parent.awaits;  // the side stream has not waited for any input yet
  for (auto& a : ch.awaits) a.done = false;
  ch.gates = parent.gates;
  ch.shard = parent.shard;
  for (auto& g : ch.gates) g.stream_done = false;
  check(cudaStreamWaitEvent(ch.s, evs[0], 0), "cudaStreamWaitEvent");
  return ch;
}

void Fork::join(Ctx& child) {
  cudaEvent_t e = get_event(parent.h, 1 + evs.size());
  check(cudaEventRecord(e, child.s), "cudaEventRecord");
  check(cudaStreamWaitEvent(parent.s, e, 0), "cudaStreamWaitEvent");
  evs.push_back(e);
  parent.ctr.mmm += child.ctr.mmm;
  parent.ctr.mvm += child.ctr.mvm;
  // the root stream now follows every use in the branch: its temporaries may go
  if (child.keep) child.keep->clear();
}

}  // namespace si
