// Native step engine: the seriesinv hot path (series_toolkit.py evaluators,
// newton_schulz.py steps, richardson.py steps) as stream-ordered sequences of
// fused FP64 GEMMs on device-resident matrices.
#pragma once
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace si {

enum Status : int { kOk = 0, kEInval = -1, kECuda = -2, kENoMem = -3 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Handle {
  std::recursive_mutex mu;  // held for the duration of every C-ABI call
  int device = 0;
  cudaMemPool_t pool = nullptr;
  static constexpr int kSide = 5;
  cudaStream_t side[kSide] = {};
  std::vector<cudaEvent_t> events;
  double* red_work = nullptr;  // reduction scratch
  size_t red_elems = 0;
  double* scalar = nullptr;    // one device double
  // live profiling of the dominant kernel (bench.py roofline): CUDA events
  // around every TMA GEMM launch, on the stream it is launched on.
  struct ProfRec {
    cudaEvent_t start, stop;
    double flops;
  };
  bool profiling = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> prof_pool;
  int64_t launches = 0;  // kernels launched by this handle
  // si_set_step_norm: device double receiving ||F'||_F^2 of the next step
  // call's residual output (one-shot: the step call consumes it)
  double* step_norm = nullptr;
  // FP64 product backend (si_set_gemm_backend): 0 = DMMA (gemm_tma.cu, the
  // default), 1 = Ozaki-II emulation on the INT8 tensor cores (ozaki.cu) for
  // products whose three dimensions are all >= oz_min_dim.
  int gemm_backend = 0;
  int oz_nmod = 16;
  int64_t oz_min_dim = 1024;
  int64_t oz_max_cols = 0;  // columns of D per emulated chunk at most (0: automatic)
  int64_t oz_max_rows = 0;  // rows of D per emulated chunk at most (0: all rows)
  int oz_variant = 0;       // INT8 kernel: 0 auto (CTA pairs), 1 CTA pairs, 2 single CTAs
  // live profiling of the INT8 tensor-core kernel inside emulated products
  std::vector<ProfRec> prof_i8;
  // Optional external allocator (si_set_allocator): the Python layer routes
  // temporaries through PyTorch's caching allocator so that one allocator owns
  // all device memory (at n=32768 a matrix is 8.6 GB; two caches do not fit).
  void* (*alloc_fn)(void* ctx, size_t bytes, void* stream) = nullptr;
  void (*free_fn)(void* ctx, void* ptr, void* stream) = nullptr;
  void* alloc_ctx = nullptr;
  // Resident-kernel programs (batched.cu) already on the device, keyed by
  // their encoded bytes: repeated launches of the same run skip the upload.
  std::unordered_map<std::string, void*> programs;
};

// Owning device buffer, released stream-ordered on its root stream (the
// stream of the C-ABI call).  Buffers created inside a concurrent branch are
// kept alive by the branch until it is joined, so their release is ordered
// after every use on the side stream.
struct Buf {
  double* p = nullptr;
  cudaStream_t free_stream = nullptr;
  Handle* h = nullptr;
  bool external = false;
  ~Buf();
};

// A matrix value: a view plus (optional) shared ownership of its storage.
// `local` (block-row sharded calls only, Ctx::shard set): the value is this
// rank's row block [r0, r1) of an n-row matrix; otherwise it is the whole
// matrix (replicated on every rank).
struct MV {
  Mat v;
  std::shared_ptr<Buf> own;
  bool local = false;
  int64_t n() const { return v.rows; }
};

struct Shard;  // shard.hpp: row split + the exchange of one sharded C-ABI call

struct Counters {
  int64_t mmm = 0, mvm = 0;
};

// Execution context for one C-ABI call: root stream + current stream.
struct Ctx {
  Handle* h;
  cudaStream_t root;
  cudaStream_t s;
  Counters ctr;
  // set on branch contexts: buffers allocated in the branch, released at join
  std::shared_ptr<std::vector<std::shared_ptr<Buf>>> keep;
  // Inputs still in flight (host->device copies): the first kernel that reads
  // one of these base pointers on this stream waits for its event first.
  struct Await {
    const void* base;
    cudaEvent_t ev;
    bool done;
  };
  std::vector<Await> awaits;
  void await_ptr(const void* p);
  // Inputs arriving in row panels (flags raised behind each panel's copy): the
  // DMMA GEMM gates its A-tile / B-slab loads per panel; every other reader
  // makes its stream wait for all panels first.
  struct Gate {
    const void* base;
    PanelWait pw;
    bool stream_done;
  };
  std::vector<Gate> gates;
  const PanelWait* gate_of(const void* p) const;
  void gate_stream(const void* p);  // stream-wait for every panel of p (once)
  // Block-row sharded execution (shard.cu): every product yields
  // this rank's rows; a replicated left / epilogue operand is read through its
  // row view, a sharded right operand is all-gathered first.
  Shard* shard = nullptr;
  // workspace of the emulated (Ozaki-II) products on a branch context, reused
  // by every product on its stream (they are stream-ordered)
  MV oz_ws;
  size_t oz_ws_bytes = 0;
  // Caller buffers this call only reads (a step's inputs, not aliased by an
  // output): the emulated products keep their operand scales + residue
  // planes across the call's products (root stream only; released with the call).
  struct Range {
    const char* base;
    size_t bytes;
  };
  std::vector<Range> stable;    // a matrix inside one of these ranges may keep its images
  std::vector<MV> stable_keep;  // engine values marked stable (kept alive for the call)
  struct OzSide;
  std::vector<std::shared_ptr<OzSide>> oz_sides;
  // Fused ||F||_F^2 of a step's residual output (si_set_step_norm,
  // newton_schulz.py:328-331): while `sq` is set, every product whose output
  // lies in [sq_lo, sq_hi) (the step's F' buffer) writes the sum-of-squares
  // slots of the values it stores (GEMM / CRT epilogue; a separate partial
  // pass on the small-n kernels) into a buffer appended here; finish_sq()
  // reduces them in product order into one device double.
  struct SqAcc {
    std::vector<std::pair<MV, int64_t>> parts;  // slot buffer, slot count
  };
  SqAcc* sq = nullptr;
  const double* sq_lo = nullptr;
  const double* sq_hi = nullptr;
  Ctx(Handle* hh, cudaStream_t st) : h(hh), root(st), s(st) {}
};

void check(cudaError_t e, const char* what);
// *out = ||F||_F^2 of the step output F: the fixed-order sum of the slots `acc`
// collected from the products that wrote F, or (no product wrote it, e.g. a
// copied F) one reduction pass over F (stream-ordered)
void finish_sq(Ctx& c, const Ctx::SqAcc& acc, const Mat& F, double* out);
// Mark an engine value that is never written again in this call as stable (its
// emulated-product operand images may be kept); it stays allocated until the
// call ends.  Root context only (no-op on branches).
void keep_stable(Ctx& c, const MV& v);
MV view(double* p, int64_t rows, int64_t cols, int64_t ld);
MV alloc(Ctx& c, int64_t rows, int64_t cols);

// D = alpha * A @ B + beta * C + diag * I  (one counted product; mv=true ticks mvm)
// `pw` (optional) gates the reads of B's row panels on arrival flags.
void gemm(Ctx& c, const MV& D, const MV& A, const MV& B, double alpha = 1.0,
          const MV* C = nullptr, double beta = 0.0, double diag = 0.0, bool mv = false,
          int64_t doff = 0, const PanelWait* pw = nullptr);
MV gemm_new(Ctx& c, const MV& A, const MV& B, double alpha = 1.0, const MV* C = nullptr,
            double beta = 0.0, double diag = 0.0, bool mv = false);
// I - X @ A
MV residual(Ctx& c, const MV& X, const MV& A);
void residual_into(Ctx& c, const MV& D, const MV& X, const MV& A);
void copy_into(Ctx& c, const MV& D, const MV& X);
MV lincomb(Ctx& c, double cdiag, const std::vector<std::pair<double, const MV*>>& terms,
           int64_t rows, int64_t cols);
// a fresh buffer shaped like x (this rank's rows of it in a sharded call)
MV alloc_like(Ctx& c, const MV& x);
// scale * I shaped like x (the identity's rows of this rank in a sharded call)
MV identity_like(Ctx& c, const MV& x, double scale = 1.0);

// ---- plans (series_toolkit.py:71-157), decoded from the int32 preorder form ----
struct PlanNode;
using PlanPtr = std::shared_ptr<const PlanNode>;
struct Instr {
  int op;  // 0 mul, 1 residual, 2 lin
  int dst, a, b;
  double cconst;
  std::vector<std::pair<double, int>> terms;
};
struct PlanNode {
  int kind;  // 0 horner, 1 split, 2 wrap, 3 table
  int h = 0, p = 0, w = 0, order = 0, nregs = 0;
  PlanPtr inner, outer;
  std::vector<Instr> prog;
};
PlanPtr decode_plan(const int32_t* code, int64_t len, const double* consts, int64_t nconsts);
int plan_order_of(const PlanNode& n);

// ---- evaluators (series_toolkit.py:263-457) ----
MV horner(Ctx& c, const MV& y, const MV& x, int h);
MV factored(Ctx& c, const MV& y, const MV& x, const MV& a, int p, int w);
MV eval_node(Ctx& c, const PlanNode& node, const MV& y, const MV& x, const MV& a);
// geometric_apply (st:432-457): `base` is plan_order(b) for the order b <= 64
// reached by repeated halving (null when that order is 1).
MV geometric(Ctx& c, const MV& y, const MV& x, int order, const MV& a, const PlanNode* base);
MV mat_pow_counted(Ctx& c, const MV& y, int e);

// ---- fork/join helpers for the executor mapping ----
struct Fork {
  Ctx& parent;
  std::vector<cudaEvent_t> evs;
  explicit Fork(Ctx& c);
  Ctx branch(int i);                 // a child ctx on side stream i, ordered after parent
  void join(Ctx& child);             // parent waits for child; counters merged
};

}  // namespace si
