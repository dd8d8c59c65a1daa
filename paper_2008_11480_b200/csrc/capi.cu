// extern "C" boundary (include/seriesinv_b200.h).  Validates arguments, maps
// exceptions to status codes, never throws across the ABI.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/seriesinv_b200.h"
#include "batched.hpp"
#include "ozaki.hpp"
#include "setup.hpp"
#include "shard.hpp"
#include "steps.hpp"

using namespace si;

struct si_handle_s {
  Handle h;
};

// A block-row communicator (SURVEY 8(b) "sharded variants that take the
// communicators created inside the handle"): the exchange plus the row split.
struct si_comm_s {
  std::unique_ptr<Exchange> ex;
  int rank = 0, world = 1;
  int64_t n = 0;
  int64_t gathers = 0, bytes_in = 0;
};

namespace {

template <typename F>
int guard(F&& f) {
  try {
    f();
    return SI_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return SI_ENOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return SI_ECUDA;
  }
}

void need(bool ok, const char* msg) {
  if (!ok) throw Error(kEInval, msg);
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

MV sq(const double* p, int64_t n) { return view(const_cast<double*>(p), n, n, n); }
MV rect(const double* p, int64_t n, int64_t r) { return view(const_cast<double*>(p), n, r, r); }

void add_counters(int64_t* counters, const Ctx& c) {
  if (counters) {
    counters[0] += c.ctr.mmm;
    counters[1] += c.ctr.mvm;
  }
}

// One C-ABI call: serialises host-side use of the handle (its side streams,
// events and profiling records) across threads -- the reference's executors
// may call in from several threads -- and sets the device.
struct Call {
  std::lock_guard<std::recursive_mutex> lock;
  Ctx c;
  int64_t* counters;
  Call(si_handle h, void* stream, int64_t* ctrs)
      : lock(h->h.mu), c(&h->h, as_stream(stream)), counters(ctrs) {
    check(cudaSetDevice(h->h.device), "cudaSetDevice");
  }
  ~Call() { add_counters(counters, c); }
};

// A step's n x n inputs that no output of the call overlaps: the emulated
// products may keep their operand images across the call (engine.cu oz_side).
// (`out_rows`: rows of each output, e.g. a rank's row block in a sharded call)
void mark_stable(Ctx& c, int64_t n, std::initializer_list<const double*> ins,
                 std::initializer_list<const double*> outs, int64_t out_rows = -1) {
  const size_t bytes = (size_t)n * (size_t)n * sizeof(double);
  const size_t obytes = (size_t)(out_rows < 0 ? n : out_rows) * (size_t)n * sizeof(double);
  for (const double* in : ins) {
    const char* a = reinterpret_cast<const char*>(in);
    bool clash = false;
    for (const double* out : outs) {
      const char* b = reinterpret_cast<const char*>(out);
      if (a < b + obytes && b < a + bytes) clash = true;
    }
    if (!clash) c.stable.push_back({a, bytes});
  }
}

// si_set_step_norm: ||F'||_F^2 of this step call's residual output F' (n x n
// at f_out), fused into the epilogues of the products that write F'
// (newton_schulz.py:328-331 reads it back as converged()); consumes the
// handle's one-shot target.  finish() after the step body.
struct StepNorm {
  Ctx& c;
  const double* f;
  int64_t n;
  double* out;
  Ctx::SqAcc acc;
  StepNorm(Call& call, const double* f_out, int64_t nn, double* target)
      : c(call.c), f(f_out), n(nn), out(target) {
    if (out) {
      c.sq = &acc;
      c.sq_lo = f;
      c.sq_hi = f + n * n;
    }
  }
  void finish() {
    c.sq = nullptr;
    if (out) finish_sq(c, acc, view(const_cast<double*>(f), n, n, n).v, out);
  }
  ~StepNorm() { c.sq = nullptr; }
};

// the handle's one-shot si_set_step_norm target, consumed first thing by
// every step call (also by one that then fails its argument checks)
double* take_step_norm(si_handle h) {
  if (!h) return nullptr;
  std::lock_guard<std::recursive_mutex> lock(h->h.mu);
  double* t = h->h.step_norm;
  h->h.step_norm = nullptr;
  return t;
}

// One sharded C-ABI call: Call + this call's Shard (row split, gather cache).
struct ShardCall {
  Call call;
  Shard sh;
  si_comm comm;
  ShardCall(si_handle h, si_comm cm, int64_t n, void* stream, int64_t* ctrs)
      : call(h, stream, ctrs), comm(cm) {
    if (!cm) throw Error(kEInval, "null communicator");
    if (n != cm->n) throw Error(kEInval, "n differs from the communicator's n");
    sh.ex = cm->ex.get();
    sh.init(n, cm->rank, cm->world);
    call.c.shard = &sh;
  }
  ~ShardCall() {
    comm->gathers += sh.gathers;
    comm->bytes_in += sh.bytes_in;
  }
  int64_t rows() const { return sh.r1 - sh.r0; }
  MV loc(const double* p, int64_t cols) {
    MV m = view(const_cast<double*>(p), rows(), cols, cols);
    m.local = true;
    return m;
  }
};

PlanPtr opt_plan(const int32_t* code, int64_t len, const double* consts, int64_t nconsts) {
  if (!code || len == 0) return nullptr;
  return decode_plan(code, len, consts, nconsts);
}

double host_fro(Ctx& c, const MV& x) {
  Handle* h = c.h;
  const size_t need_elems = reduce_work_elems(x.v);
  if (h->red_elems < need_elems) {
    if (h->red_work) cudaFree(h->red_work);
    h->red_work = nullptr;
    check(cudaMalloc(&h->red_work, need_elems * sizeof(double)), "cudaMalloc");
    h->red_elems = need_elems;
  }
  check(launch_sumsq(x.v, h->scalar, h->red_work, c.s), "sumsq");
  double v = 0.0;
  check(cudaMemcpyAsync(&v, h->scalar, sizeof(double), cudaMemcpyDeviceToHost, c.s), "memcpy");
  check(cudaStreamSynchronize(c.s), "sync");
  return std::sqrt(v);
}

// series_toolkit.py:270-276 -- Y = I - X A, checked against a supplied Y.
MV formed_y(Ctx& c, const double* y, const MV& x, const MV& a) {
  MV ye = residual(c, x, a);
  if (y) {
    MV yv = sq(y, x.v.rows);
    MV diff = lincomb(c, 0.0, {{1.0, &ye}, {-1.0, &yv}}, x.v.rows, x.v.cols);
    const double gap = host_fro(c, diff);
    const double ny = host_fro(c, yv);
    if (gap > 1e-10 * (1.0 + ny)) throw Error(kEInval, "supplied Y does not match I - X A");
  }
  return ye;
}

}  // namespace

extern "C" {

int si_version(void) { return 1; }
const char* si_last_error(void) { return get_error(); }

int si_create(int device, si_handle* out) {
  return guard([&] {
    need(out != nullptr, "null handle pointer");
    check(cudaSetDevice(device), "cudaSetDevice");
    auto* hs = new si_handle_s();
    hs->h.device = device;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    check(cudaMemPoolCreate(&hs->h.pool, &props), "cudaMemPoolCreate");
    uint64_t thresh = UINT64_MAX;
    check(cudaMemPoolSetAttribute(hs->h.pool, cudaMemPoolAttrReleaseThreshold, &thresh),
          "cudaMemPoolSetAttribute");
    for (int i = 0; i < Handle::kSide; ++i)
      check(cudaStreamCreateWithFlags(&hs->h.side[i], cudaStreamNonBlocking), "cudaStreamCreate");
    check(cudaMalloc(&hs->h.scalar, sizeof(double)), "cudaMalloc");
    *out = hs;
  });
}

int si_destroy(si_handle h) {
  return guard([&] {
    if (!h) return;
    cudaSetDevice(h->h.device);
    cudaDeviceSynchronize();
    for (auto e : h->h.events) cudaEventDestroy(e);
    for (int i = 0; i < Handle::kSide; ++i)
      if (h->h.side[i]) cudaStreamDestroy(h->h.side[i]);
    if (h->h.red_work) cudaFree(h->h.red_work);
    if (h->h.scalar) cudaFree(h->h.scalar);
    for (auto& kv : h->h.programs) cudaFree(kv.second);
    if (h->h.pool) cudaMemPoolDestroy(h->h.pool);
    delete h;
  });
}

int si_set_step_norm(si_handle h, double* fro2) {
  return guard([&] {
    need(h != nullptr, "null handle");
    std::lock_guard<std::recursive_mutex> lock(h->h.mu);
    h->h.step_norm = fro2;
  });
}

int si_set_allocator(si_handle h, void* (*alloc_fn)(void*, size_t, void*),
                     void (*free_fn)(void*, void*, void*), void* ctx) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need((alloc_fn == nullptr) == (free_fn == nullptr), "alloc_fn and free_fn go together");
    h->h.alloc_fn = alloc_fn;
    h->h.free_fn = free_fn;
    h->h.alloc_ctx = ctx;
  });
}

int si_trim(si_handle h) {
  return guard([&] {
    need(h != nullptr, "null handle");
    check(cudaDeviceSynchronize(), "sync");
    check(cudaMemPoolTrimTo(h->h.pool, 0), "cudaMemPoolTrimTo");
  });
}

int si_gemm(si_handle h, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
            int64_t lda, const double* B, int64_t ldb, double beta, const double* C, int64_t ldc,
            double diag, double* D, int64_t ldd, int is_mv, int64_t* counters, void* stream) {
  return si_gemm_ex(h, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, diag, 0, D, ldd, is_mv,
                    counters, stream);
}

int si_gemm_ex(si_handle h, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
               int64_t lda, const double* B, int64_t ldb, double beta, const double* C,
               int64_t ldc, double diag, int64_t diag_offset, double* D, int64_t ldd, int is_mv,
               int64_t* counters, void* stream) {
  return guard([&] {
    // empty operands may be NULL (numpy / torch give empty arrays no storage)
    need(h && (A || m * k == 0) && (B || k * n == 0) && (D || m * n == 0), "null pointer");
    need(m >= 0 && n >= 0 && k >= 0, "negative dimension");
    need(lda >= k && ldb >= n && ldd >= n, "leading dimension too small");
    need(beta == 0.0 || m * n == 0 || (C && ldc >= n), "beta != 0 needs C");
    Call call(h, stream, counters);
    MV a = view(const_cast<double*>(A), m, k, lda), b = view(const_cast<double*>(B), k, n, ldb);
    MV d = view(D, m, n, ldd);
    MV cm = view(const_cast<double*>(C), m, n, ldc);
    gemm(call.c, d, a, b, alpha, C ? &cm : nullptr, beta, diag, is_mv != 0, diag_offset);
  });
}

int si_gemm_panels(si_handle h, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                   int64_t lda, const double* B, int64_t ldb, double beta, const double* C,
                   int64_t ldc, double diag, int64_t diag_offset, double* D, int64_t ldd,
                   const uint32_t* ready_flags, uint32_t epoch, const int64_t* panel_bounds,
                   int npanels, int is_mv, int64_t* counters, void* stream) {
  return guard([&] {
    need(h && (A || m * k == 0) && (B || k * n == 0) && (D || m * n == 0), "null pointer");
    need(m >= 0 && n >= 0 && k >= 0, "negative dimension");
    need(lda >= k && ldb >= n && ldd >= n, "leading dimension too small");
    need(beta == 0.0 || m * n == 0 || (C && ldc >= n), "beta != 0 needs C");
    need(npanels >= 0 && npanels <= kMaxPanels, "npanels out of range");
    need(npanels == 0 || (ready_flags && panel_bounds), "null panel arrays");
    PanelWait pw;
    pw.ready = ready_flags;
    pw.epoch = epoch;
    pw.npanels = npanels;
    if (npanels > 0) {  // npanels == 0 is the ungated product; its arrays may be NULL
      for (int p = 0; p <= npanels; ++p) {
        need(panel_bounds[p] >= 0 && panel_bounds[p] <= k, "panel bound out of range");
        need(p == 0 || panel_bounds[p] >= panel_bounds[p - 1], "panel bounds not ascending");
        pw.bounds[p] = (int)panel_bounds[p];
      }
      need(panel_bounds[0] == 0 && panel_bounds[npanels] == k,
           "panels must cover the k rows of B");
    }
    Call call(h, stream, counters);
    MV a = view(const_cast<double*>(A), m, k, lda), b = view(const_cast<double*>(B), k, n, ldb);
    MV d = view(D, m, n, ldd);
    MV cm = view(const_cast<double*>(C), m, n, ldc);
    gemm(call.c, d, a, b, alpha, C ? &cm : nullptr, beta, diag, is_mv != 0, diag_offset, &pw);
  });
}

int si_sym_alloc(si_handle h, size_t bytes, void** ptr, unsigned char handle_out[64]) {
  return guard([&] {
    need(h && ptr && handle_out, "null pointer");
    need(bytes > 0, "empty allocation");
    check(cudaSetDevice(h->h.device), "cudaSetDevice");
    void* p = nullptr;
    const cudaError_t err = cudaMalloc(&p, bytes);
    if (err == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      throw Error(kENoMem, "cudaMalloc of an exchange buffer failed");
    }
    check(err, "cudaMalloc");
    check(cudaMemset(p, 0, bytes), "cudaMemset");
    check(cudaDeviceSynchronize(), "sync");  // zeroed before any peer or stream sees it
    cudaIpcMemHandle_t ipc;
    const cudaError_t e2 = cudaIpcGetMemHandle(&ipc, p);
    if (e2 != cudaSuccess) {
      cudaFree(p);
      check(e2, "cudaIpcGetMemHandle");
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    std::memcpy(handle_out, &ipc, 64);
    *ptr = p;
  });
}

int si_sym_free(si_handle h, void* ptr) {
  return guard([&] {
    need(h != nullptr, "null handle");
    if (!ptr) return;
    check(cudaSetDevice(h->h.device), "cudaSetDevice");
    check(cudaDeviceSynchronize(), "sync");
    check(cudaFree(ptr), "cudaFree");
  });
}

int si_sym_open(si_handle h, const unsigned char handle[64], void** ptr) {
  return guard([&] {
    need(h && handle && ptr, "null pointer");
    check(cudaSetDevice(h->h.device), "cudaSetDevice");
    cudaIpcMemHandle_t ipc;
    std::memcpy(&ipc, handle, 64);
    check(cudaIpcOpenMemHandle(ptr, ipc, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

int si_sym_close(si_handle h, void* ptr) {
  return guard([&] {
    need(h != nullptr, "null handle");
    if (!ptr) return;
    check(cudaSetDevice(h->h.device), "cudaSetDevice");
    check(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
  });
}

int si_stream_write_u32(si_handle h, uint32_t* addr, uint32_t value, void* stream) {
  return guard([&] {
    need(h && addr, "null pointer");
    Call call(h, stream, nullptr);
    check(stream_write_u32(addr, value, call.c.s), "stream write");
  });
}

int si_stream_wait_u32(si_handle h, const uint32_t* addr, uint32_t value, void* stream) {
  return guard([&] {
    need(h && addr, "null pointer");
    Call call(h, stream, nullptr);
    check(stream_wait_u32(addr, value, call.c.s), "stream wait");
  });
}

int si_copy_async(si_handle h, void* dst, const void* src, size_t bytes, void* stream) {
  return guard([&] {
    need(h && (bytes == 0 || (dst && src)), "null pointer");
    Call call(h, stream, nullptr);
    if (bytes) check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, call.c.s), "copy");
  });
}

int si_lincomb(si_handle h, int64_t m, int64_t n, double cdiag, int nterms, const double* coefs,
               const double* const* X, const int64_t* ldx, double* D, int64_t ldd, void* stream) {
  return si_lincomb_ex(h, m, n, cdiag, 0, nterms, coefs, X, ldx, D, ldd, stream);
}

int si_lincomb_ex(si_handle h, int64_t m, int64_t n, double cdiag, int64_t diag_offset,
                  int nterms, const double* coefs, const double* const* X, const int64_t* ldx,
                  double* D, int64_t ldd, void* stream) {
  return guard([&] {
    need(h && D, "null pointer");
    need(nterms >= 0 && nterms <= kMaxLinTerms, "nterms out of range");
    need(nterms == 0 || (coefs && X && ldx), "null term arrays");
    Call call(h, stream, nullptr);
    Mat xs[kMaxLinTerms];
    for (int i = 0; i < nterms; ++i) {
      need(X[i] != nullptr && ldx[i] >= n, "bad term");
      xs[i] = view(const_cast<double*>(X[i]), m, n, ldx[i]).v;
    }
    Mat d = view(D, m, n, ldd).v;
    check(launch_lincomb(d, cdiag, diag_offset, nterms, coefs, xs, call.c.s), "lincomb");
    h->h.launches += 1;
  });
}

int si_fro_norm(si_handle h, int64_t m, int64_t n, const double* X, int64_t ldx, double* out,
                void* stream) {
  return guard([&] {
    need(h && X && out, "null pointer");
    Call call(h, stream, nullptr);
    *out = host_fro(call.c, view(const_cast<double*>(X), m, n, ldx));
  });
}

int si_inf_norm(si_handle h, int64_t m, int64_t n, const double* X, int64_t ldx, double* out,
                void* stream) {
  return guard([&] {
    need(h && X && out, "null pointer");
    Call call(h, stream, nullptr);
    Handle* hh = &h->h;
    Mat x = view(const_cast<double*>(X), m, n, ldx).v;
    const size_t ne = reduce_work_elems(x);
    if (hh->red_elems < ne) {
      if (hh->red_work) cudaFree(hh->red_work);
      hh->red_work = nullptr;
      check(cudaMalloc(&hh->red_work, ne * sizeof(double)), "cudaMalloc");
      hh->red_elems = ne;
    }
    check(launch_inf_norm(x, hh->scalar, hh->red_work, call.c.s), "inf_norm");
    check(cudaMemcpyAsync(out, hh->scalar, sizeof(double), cudaMemcpyDeviceToHost, call.c.s),
          "memcpy");
    check(cudaStreamSynchronize(call.c.s), "sync");
  });
}

int si_split_scalar(si_handle h, int64_t n, const double* A, double alpha, double* precond,
                    double* residual, void* stream) {
  return guard([&] {
    need(h && A && residual, "null pointer");
    need(n >= 1 && alpha > 0.0, "bad splitting arguments");
    Call call(h, stream, nullptr);
    Mat p = view(precond, n, n, n).v, b = view(residual, n, n, n).v;
    check(launch_scalar_split(p, b, sq(A, n).v, alpha, call.c.s), "split_scalar");
  });
}

int si_split_diagonal(si_handle h, int64_t n, const double* A, double* precond, double* residual,
                      void* stream) {
  return guard([&] {
    need(h && A && residual, "null pointer");
    Call call(h, stream, nullptr);
    Mat p = view(precond, n, n, n).v, b = view(residual, n, n, n).v;
    check(launch_diag_split(p, b, sq(A, n).v, call.c.s), "split_diagonal");
  });
}

int si_symmetrize(si_handle h, int64_t n, const double* A, double* out, void* stream) {
  return guard([&] {
    need(h && A && out && A != out, "bad pointer");
    Call call(h, stream, nullptr);
    Mat d = view(out, n, n, n).v;
    check(launch_symmetrize(d, sq(A, n).v, call.c.s), "symmetrize");
  });
}

int si_symmetrize_checked(si_handle h, int64_t n, const double* A, double* out, double* asym_fro,
                          double* fro, double* nonfinite, void* stream) {
  return guard([&] {
    need(h && A && out && asym_fro && fro && nonfinite, "null pointer");
    need(n >= 0, "negative dimension");
    Call call(h, stream, nullptr);
    if (n == 0) {
      *asym_fro = *fro = *nonfinite = 0.0;
      return;
    }
    MV work = alloc(call.c, 1, (int64_t)symcheck_work_elems() + 3);
    double* res = work.v.p + symcheck_work_elems();
    Mat d = view(out, n, n, n).v;
    check(launch_symcheck(d, sq(A, n).v, work.v.p, res, call.c.s), "symcheck");
    h->h.launches += 2;
    double host[3];
    check(cudaMemcpyAsync(host, res, sizeof(host), cudaMemcpyDeviceToHost, call.c.s), "memcpy");
    check(cudaStreamSynchronize(call.c.s), "sync");
    *asym_fro = host[0];
    *fro = host[1];
    *nonfinite = host[2];
  });
}

int si_is_positive_definite(si_handle h, int64_t n, const double* A, int64_t lda,
                            double pivot_tol, int default_tol, int* is_pd, int64_t* fail_index,
                            double* fail_pivot, void* stream) {
  return guard([&] {
    need(h && (A || n == 0) && is_pd, "null pointer");
    need(n >= 0 && lda >= n, "bad dimensions");
    Call call(h, stream, nullptr);
    int64_t idx = -1;
    double piv = 0.0;
    *is_pd = cholesky_pd(call.c, view(const_cast<double*>(A), n, n, lda), pivot_tol,
                         default_tol != 0, &idx, &piv)
                 ? 1
                 : 0;
    if (fail_index) *fail_index = idx;
    if (fail_pivot) *fail_pivot = piv;
  });
}

int si_power_iterate(si_handle h, int64_t n, const double* A, int64_t lda, double* x,
                     double tol, int64_t max_iter, int check_every, double* est, double* best,
                     int64_t* iters, int* status, void* stream) {
  return guard([&] {
    need(h && A && x && est && best && iters && status, "null pointer");
    need(n >= 1 && lda >= n && max_iter >= 1 && check_every >= 1, "bad arguments");
    Call call(h, stream, nullptr);
    const int np = sumsq_partials();
    // y, partial sums, and the PowerState (as doubles)
    MV work = alloc(call.c, 1, n + np + 8);
    double* y = work.v.p;
    double* part = y + n;
    PowerState* st = reinterpret_cast<PowerState*>(part + np);
    check(cudaMemsetAsync(st, 0, sizeof(PowerState), call.c.s), "memset");
    PowerState hs{};
    Mat a = view(const_cast<double*>(A), n, n, lda).v;
    int64_t queued = 0;
    while (queued < max_iter) {
      const int k = (int)std::min<int64_t>(check_every, max_iter - queued);
      check(launch_power_iters(a, x, y, part, st, tol, max_iter, k, call.c.s), "power iteration");
      h->h.launches += 3 * k;
      queued += k;
      check(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, call.c.s), "memcpy");
      check(cudaStreamSynchronize(call.c.s), "sync");
      if (hs.status != kPowerRunning) break;
    }
    *est = hs.est;
    *best = hs.best;
    *iters = hs.iters;
    *status = hs.status;
  });
}

int si_horner_eval(si_handle h, int64_t n, const double* y, const double* x, int order,
                   const double* a, int form_y, double* out, int64_t* counters, void* stream) {
  return guard([&] {
    need(h && x && out, "null pointer");
    need(order >= 1, "order h must be >= 1");
    need(!form_y || a, "form_y=True requires the matrix a");
    need(form_y || y, "y is required unless form_y=True");
    Call call(h, stream, counters);
    MV xv = sq(x, n);
    MV yv = form_y ? formed_y(call.c, y, xv, sq(a, n)) : sq(y, n);
    copy_into(call.c, sq(out, n), horner(call.c, yv, xv, order));
  });
}

int si_factored_eval(si_handle h, int64_t n, const double* y, const double* x, const double* a,
                     int p, int w, int form_y, double* out, int64_t* counters, void* stream) {
  return guard([&] {
    need(h && x && a && out, "null pointer");
    need(p >= 0 && w >= 1, "requires p >= 0 and w >= 1");
    need(form_y || y, "y is required unless form_y=True");
    Call call(h, stream, counters);
    MV xv = sq(x, n), av = sq(a, n);
    MV yv = form_y ? formed_y(call.c, y, xv, av) : sq(y, n);
    copy_into(call.c, sq(out, n), factored(call.c, yv, xv, av, p, w));
  });
}

int si_nested_eval(si_handle h, int64_t n, const double* y, const double* x, const double* a,
                   const int32_t* plan, int64_t plan_len, const double* consts, int64_t nconsts,
                   int form_y, double* out, int64_t* counters, void* stream) {
  return guard([&] {
    need(h && x && a && out, "null pointer");
    need(form_y || y, "y is required unless form_y=True");
    PlanPtr pl = decode_plan(plan, plan_len, consts, nconsts);
    Call call(h, stream, counters);
    MV xv = sq(x, n), av = sq(a, n);
    MV yv = form_y ? formed_y(call.c, y, xv, av) : sq(y, n);
    copy_into(call.c, sq(out, n), eval_node(call.c, *pl, yv, xv, av));
  });
}

int si_geometric_apply(si_handle h, int64_t n, const double* y, const double* x, int order,
                       const double* a, const int32_t* base_plan, int64_t plan_len,
                       const double* consts, int64_t nconsts, double* out, int64_t* counters,
                       void* stream) {
  return guard([&] {
    need(h && y && x && a && out, "null pointer");
    need(order >= 1, "order must be >= 1");
    PlanPtr pl = opt_plan(base_plan, plan_len, consts, nconsts);
    Call call(h, stream, counters);
    copy_into(call.c, sq(out, n), geometric(call.c, sq(y, n), sq(x, n), order, sq(a, n), pl.get()));
  });
}

int si_mat_pow_counted(si_handle h, int64_t n, const double* y, int e, double* out,
                       int64_t* counters, void* stream) {
  return guard([&] {
    need(h && y && out, "null pointer");
    need(e >= 0, "exponent must be non-negative");
    Call call(h, stream, counters);
    copy_into(call.c, sq(out, n), mat_pow_counted(call.c, sq(y, n), e));
  });
}

int si_initial_series(si_handle h, int64_t n, const double* precond, const double* residual,
                      const double* a, int p, int w, double* g_out, double* f_out,
                      int64_t* counters, void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && precond && residual && a && g_out && f_out, "null pointer");
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    initial_series(call.c, sq(precond, n), sq(residual, n), sq(a, n), p, w, sq(g_out, n),
                   sq(f_out, n));
    norm.finish();
  });
}

int si_ns_step(si_handle h, int64_t n, const double* a, const double* g, const double* f,
               int order, const int32_t* plan, int64_t plan_len, const double* consts,
               int64_t nconsts, double* g_out, double* f_out, int64_t* counters, void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && a && g && f && g_out && f_out, "null pointer");
    PlanPtr pl = opt_plan(plan, plan_len, consts, nconsts);
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    mark_stable(call.c, n, {a, g, f}, {g_out, f_out});
    ns_step(call.c, sq(a, n), sq(g, n), sq(f, n), order, pl.get(), sq(g_out, n), sq(f_out, n));
    norm.finish();
  });
}

int si_ns_step_ex(si_handle h, int64_t n, const double* a, const double* g, const double* f,
                  int order, const int32_t* plan, int64_t plan_len, const double* consts,
                  int64_t nconsts, void* const* input_ready_events, void* g_done_event,
                  double* g_out, double* f_out, int64_t* counters, void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && a && g && f && g_out && f_out, "null pointer");
    PlanPtr pl = opt_plan(plan, plan_len, consts, nconsts);
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    mark_stable(call.c, n, {a, g, f}, {g_out, f_out});
    if (input_ready_events) {
      const double* bases[3] = {a, g, f};
      for (int i = 0; i < 3; ++i)
        if (input_ready_events[i])
          call.c.awaits.push_back({bases[i], reinterpret_cast<cudaEvent_t>(input_ready_events[i]),
                                   false});
    }
    ns_step(call.c, sq(a, n), sq(g, n), sq(f, n), order, pl.get(), sq(g_out, n), sq(f_out, n),
            reinterpret_cast<cudaEvent_t>(g_done_event));
    norm.finish();
  });
}

int si_ns_step_gated(si_handle h, int64_t n, const double* a, const double* g, const double* f,
                     int order, const int32_t* plan, int64_t plan_len, const double* consts,
                     int64_t nconsts, const uint32_t* input_flags, uint32_t epoch, int npanels,
                     void* g_done_event, void* const* f_chunk_events, int f_chunks,
                     double* g_out, double* f_out, int64_t* counters, void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && a && g && f && g_out && f_out, "null pointer");
    need(!input_flags || (npanels >= 1 && npanels <= kMaxPanels), "npanels out of range");
    need(f_chunks >= 0 && (f_chunks == 0 || f_chunk_events), "bad f_chunks");
    PlanPtr pl = opt_plan(plan, plan_len, consts, nconsts);
    std::vector<cudaEvent_t> chunks(f_chunks);
    for (int k = 0; k < f_chunks; ++k) chunks[k] = reinterpret_cast<cudaEvent_t>(f_chunk_events[k]);
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    mark_stable(call.c, n, {a, g, f}, {g_out, f_out});
    if (input_flags) {
      const double* bases[3] = {a, g, f};
      for (int i = 0; i < 3; ++i) {
        Ctx::Gate gt{};
        gt.base = bases[i];
        gt.pw.ready = input_flags + kMaxPanels * i;
        gt.pw.epoch = epoch;
        gt.pw.npanels = npanels;
        for (int p = 0; p <= npanels; ++p) gt.pw.bounds[p] = (int)(n * p / npanels);
        gt.stream_done = false;
        call.c.gates.push_back(gt);
      }
    }
    ns_step(call.c, sq(a, n), sq(g, n), sq(f, n), order, pl.get(), sq(g_out, n), sq(f_out, n),
            reinterpret_cast<cudaEvent_t>(g_done_event), f_chunks,
            f_chunks ? chunks.data() : nullptr);
    norm.finish();
  });
}

int si_composite_step(si_handle h, int64_t n, const double* a, const double* g, const double* f,
                      const double* precond, const double* residual, const double* split_matrix,
                      int nrates, const int32_t* rates, const int32_t* plans,
                      const int64_t* plan_offsets, const double* consts, int64_t nconsts,
                      int order_n, int concurrent, double* g_out, double* f_out,
                      int64_t* counters, void* stream) {
  return si_composite_step_ex(h, n, a, g, f, precond, residual, split_matrix, nrates, rates, plans,
                              plan_offsets, consts, nconsts, order_n, concurrent, nullptr,
                              nullptr, g_out, f_out, counters, stream);
}

int si_composite_step_ex(si_handle h, int64_t n, const double* a, const double* g,
                         const double* f, const double* precond, const double* residual,
                         const double* split_matrix, int nrates, const int32_t* rates,
                         const int32_t* plans, const int64_t* plan_offsets, const double* consts,
                         int64_t nconsts, int order_n, int concurrent,
                         void* const* input_ready_events, void* g_done_event, double* g_out,
                         double* f_out, int64_t* counters, void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && a && g && f && precond && residual && split_matrix && g_out && f_out,
         "null pointer");
    need(nrates >= 1 && rates, "composite spec needs at least one rate");
    need(order_n >= 1, "order_n must be >= 1");
    std::vector<int> rv(rates, rates + nrates);
    std::vector<PlanPtr> owned(nrates);
    std::vector<const PlanNode*> pv(nrates, nullptr);
    for (int i = 0; i < nrates; ++i) {
      need(rv[i] >= 1, "rates must be positive integers");
      if (plans && plan_offsets && plan_offsets[i + 1] > plan_offsets[i]) {
        owned[i] = decode_plan(plans + plan_offsets[i], plan_offsets[i + 1] - plan_offsets[i],
                               consts, nconsts);
        pv[i] = owned[i].get();
      }
    }
    StepEvents ev;
    if (input_ready_events)
      for (int i = 0; i < StepEvents::kInputs; ++i)
        ev.ready[i] = reinterpret_cast<cudaEvent_t>(input_ready_events[i]);
    ev.g_done = reinterpret_cast<cudaEvent_t>(g_done_event);
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    mark_stable(call.c, n, {a, g, f, precond, residual, split_matrix}, {g_out, f_out});
    composite_step(call.c, sq(a, n), sq(g, n), sq(f, n), sq(precond, n), sq(residual, n),
                   sq(split_matrix, n), rv, pv, order_n, concurrent != 0, sq(g_out, n),
                   sq(f_out, n), &ev);
    norm.finish();
  });
}

int si_composite_step_gated(si_handle h, int64_t n, const double* a, const double* g,
                            const double* f, const double* precond, const double* residual,
                            const double* split_matrix, int nrates, const int32_t* rates,
                            const int32_t* plans, const int64_t* plan_offsets,
                            const double* consts, int64_t nconsts, int order_n, int concurrent,
                            const uint32_t* input_flags, uint32_t epoch, int npanels,
                            void* g_done_event, void* const* f_chunk_events, int f_chunks,
                            double* g_out, double* f_out, int64_t* counters, void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && a && g && f && precond && residual && split_matrix && g_out && f_out,
         "null pointer");
    need(nrates >= 1 && rates, "composite spec needs at least one rate");
    need(order_n >= 1, "order_n must be >= 1");
    need(!input_flags || (npanels >= 1 && npanels <= kMaxPanels), "npanels out of range");
    need(f_chunks >= 0 && (f_chunks == 0 || f_chunk_events), "bad f_chunks");
    std::vector<int> rv(rates, rates + nrates);
    std::vector<PlanPtr> owned(nrates);
    std::vector<const PlanNode*> pv(nrates, nullptr);
    for (int i = 0; i < nrates; ++i) {
      need(rv[i] >= 1, "rates must be positive integers");
      if (plans && plan_offsets && plan_offsets[i + 1] > plan_offsets[i]) {
        owned[i] = decode_plan(plans + plan_offsets[i], plan_offsets[i + 1] - plan_offsets[i],
                               consts, nconsts);
        pv[i] = owned[i].get();
      }
    }
    StepEvents ev;
    ev.g_done = reinterpret_cast<cudaEvent_t>(g_done_event);
    std::vector<cudaEvent_t> chunks(f_chunks);
    for (int k = 0; k < f_chunks; ++k) chunks[k] = reinterpret_cast<cudaEvent_t>(f_chunk_events[k]);
    ev.f_chunk = f_chunks ? chunks.data() : nullptr;
    ev.f_chunks = f_chunks;
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    mark_stable(call.c, n, {a, g, f, precond, residual, split_matrix}, {g_out, f_out});
    if (input_flags) {
      const double* bases[6] = {a, g, f, precond, residual, split_matrix};
      for (int i = 0; i < 6; ++i) {
        Ctx::Gate gt{};
        gt.base = bases[i];
        gt.pw.ready = input_flags + kMaxPanels * i;
        gt.pw.epoch = epoch;
        gt.pw.npanels = npanels;
        for (int p = 0; p <= npanels; ++p) gt.pw.bounds[p] = (int)(n * p / npanels);
        gt.stream_done = false;
        call.c.gates.push_back(gt);
      }
    }
    composite_step(call.c, sq(a, n), sq(g, n), sq(f, n), sq(precond, n), sq(residual, n),
                   sq(split_matrix, n), rv, pv, order_n, concurrent != 0, sq(g_out, n),
                   sq(f_out, n), &ev);
    norm.finish();
  });
}

int si_composite_parts(si_handle h, int64_t n, const double* a, const double* precond,
                       const double* residual, const double* split_matrix, int nrates,
                       const int32_t* rates, const int32_t* plans, const int64_t* plan_offsets,
                       const double* consts, int64_t nconsts, double* t_out, double* r_out,
                       int64_t* counters, void* stream) {
  return guard([&] {
    need(h && a && precond && residual && split_matrix && t_out && r_out, "null pointer");
    need(nrates >= 1 && rates, "composite spec needs at least one rate");
    std::vector<int> rv(rates, rates + nrates);
    std::vector<PlanPtr> owned(nrates);
    std::vector<const PlanNode*> pv(nrates, nullptr);
    for (int i = 0; i < nrates; ++i) {
      need(rv[i] >= 1, "rates must be positive integers");
      if (plans && plan_offsets && plan_offsets[i + 1] > plan_offsets[i]) {
        owned[i] = decode_plan(plans + plan_offsets[i], plan_offsets[i + 1] - plan_offsets[i],
                               consts, nconsts);
        pv[i] = owned[i].get();
      }
    }
    Call call(h, stream, counters);
    composite_parts(call.c, sq(a, n), sq(precond, n), sq(residual, n), sq(split_matrix, n), rv, pv,
                    sq(t_out, n), sq(r_out, n));
  });
}

int si_composite_apply(si_handle h, int64_t n, const double* a, const double* g, const double* f,
                       const double* t, const double* r, int order_n, double* g_out,
                       double* f_out, int64_t* counters, void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && a && g && f && t && r && g_out && f_out, "null pointer");
    need(order_n >= 1, "order_n must be >= 1");
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    composite_apply(call.c, sq(a, n), sq(g, n), sq(f, n), sq(t, n), sq(r, n), order_n,
                    sq(g_out, n), sq(f_out, n));
    norm.finish();
  });
}

int si_initial_double(si_handle h, int64_t n, const double* precond, const double* residual,
                      const double* a, int p, int w, int order, double* g_out, double* f_out,
                      double* l_out, double* r_out, int64_t* counters, void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && precond && residual && a && g_out && f_out && l_out && r_out, "null pointer");
    need(order >= 1, "order must be >= 1");
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    initial_double(call.c, sq(precond, n), sq(residual, n), sq(a, n), p, w, order, sq(g_out, n),
                   sq(f_out, n), sq(l_out, n), sq(r_out, n));
    norm.finish();
  });
}

int si_double_ns_step(si_handle h, int64_t n, const double* a, const double* g, const double* f,
                      const double* l, const double* r, int order, int concurrent, double* g_out,
                      double* f_out, double* l_out, double* r_out, int64_t* counters,
                      void* stream) {
  return guard([&] {
    double* fro2 = take_step_norm(h);
    need(h && a && g && f && l && r && g_out && f_out && l_out && r_out, "null pointer");
    Call call(h, stream, counters);
    StepNorm norm(call, f_out, n, fro2);
    double_ns_step(call.c, sq(a, n), sq(g, n), sq(f, n), sq(l, n), sq(r, n), order,
                   concurrent != 0, sq(g_out, n), sq(f_out, n), sq(l_out, n), sq(r_out, n));
    norm.finish();
  });
}

int si_additive_correction_step(si_handle h, int64_t n, const double* a, const double* z,
                                const double* g, int p, double* z_out, double* g_out,
                                int64_t* counters, void* stream) {
  return guard([&] {
    need(h && a && z && g && z_out && g_out, "null pointer");
    Call call(h, stream, counters);
    additive_correction_step(call.c, sq(a, n), sq(z, n), sq(g, n), p, sq(z_out, n),
                             sq(g_out, n));
  });
}

int si_richardson_step(si_handle h, int64_t n, int64_t nrhs, const double* a, const double* b,
                       const double* theta, const double* g, const double* f, const double* l,
                       const double* r, int order, int q, double* g_out, double* f_out,
                       double* l_out, double* r_out, double* theta_out, int64_t* counters,
                       void* stream) {
  return guard([&] {
    need(h && a && b && theta && g && f && l && r && g_out && f_out && l_out && r_out &&
             theta_out,
         "null pointer");
    need(nrhs >= 1, "nrhs must be >= 1");
    Call call(h, stream, counters);
    richardson_step(call.c, sq(a, n), rect(b, n, nrhs), rect(theta, n, nrhs), sq(g, n), sq(f, n),
                    sq(l, n), sq(r, n), order, q, sq(g_out, n), sq(f_out, n), sq(l_out, n),
                    sq(r_out, n), rect(theta_out, n, nrhs));
  });
}

namespace {
int recursive_step_impl(si_handle h, int64_t n, int64_t nrhs, const double* a, const double* b,
                        const double* theta, const double* g, const double* f, const double* l,
                        const double* r, const double* omega, const double* ns_part, int order,
                        const int32_t* factor_plan, int64_t plan_len, const double* consts,
                        int64_t nconsts, int doubling_sum, int concurrent,
                        void* const* input_ready_events, void* const* output_done_events,
                        double* g_out, double* f_out, double* l_out, double* r_out,
                        double* omega_out, double* ns_out, double* theta_out, int64_t* counters,
                        void* stream) {
  return guard([&] {
    need(h && a && b && theta && g && f && l && r && g_out && f_out && l_out && r_out &&
             omega_out && ns_out && theta_out,
         "null pointer");
    need(nrhs >= 1, "nrhs must be >= 1");
    PlanPtr pl = opt_plan(factor_plan, plan_len, consts, nconsts);
    if (pl) need(plan_order_of(*pl) == order, "factor plan order != iteration order");
    Call call(h, stream, counters);
    if (input_ready_events) {
      const double* bases[9] = {a, b, theta, g, f, l, r, omega, ns_part};
      for (int i = 0; i < 9; ++i)
        if (input_ready_events[i] && bases[i])
          call.c.awaits.push_back({bases[i], reinterpret_cast<cudaEvent_t>(input_ready_events[i]),
                                   false});
    }
    cudaEvent_t done[kRecOutputs] = {};
    if (output_done_events)
      for (int i = 0; i < kRecOutputs; ++i)
        done[i] = reinterpret_cast<cudaEvent_t>(output_done_events[i]);
    MV om = omega ? sq(omega, n) : MV{}, nsp = ns_part ? sq(ns_part, n) : MV{};
    richardson_recursive_step(call.c, sq(a, n), rect(b, n, nrhs), rect(theta, n, nrhs), sq(g, n),
                              sq(f, n), sq(l, n), sq(r, n), omega ? &om : nullptr,
                              ns_part ? &nsp : nullptr, order, concurrent != 0, pl.get(),
                              doubling_sum != 0, sq(g_out, n), sq(f_out, n), sq(l_out, n),
                              sq(r_out, n), sq(omega_out, n), sq(ns_out, n),
                              rect(theta_out, n, nrhs), output_done_events ? done : nullptr);
    // inputs the DAG did not read (g, f in the steady state) are part of the
    // call's state all the same: the stream does not leave the call before
    // their copies have landed
    for (auto& aw : call.c.awaits)
      if (!aw.done) {
        check(cudaStreamWaitEvent(call.c.s, aw.ev, 0), "cudaStreamWaitEvent");
        aw.done = true;
      }
  });
}
}  // namespace

int si_richardson_recursive_step(si_handle h, int64_t n, int64_t nrhs, const double* a,
                                 const double* b, const double* theta, const double* g,
                                 const double* f, const double* l, const double* r,
                                 const double* omega, const double* ns_part, int order,
                                 const int32_t* factor_plan, int64_t plan_len,
                                 const double* consts, int64_t nconsts, int doubling_sum,
                                 int concurrent, double* g_out, double* f_out, double* l_out,
                                 double* r_out, double* omega_out, double* ns_out,
                                 double* theta_out, int64_t* counters, void* stream) {
  return recursive_step_impl(h, n, nrhs, a, b, theta, g, f, l, r, omega, ns_part, order,
                             factor_plan, plan_len, consts, nconsts, doubling_sum, concurrent,
                             nullptr, nullptr, g_out, f_out, l_out, r_out, omega_out, ns_out,
                             theta_out, counters, stream);
}

int si_richardson_recursive_step_ex(si_handle h, int64_t n, int64_t nrhs, const double* a,
                                    const double* b, const double* theta, const double* g,
                                    const double* f, const double* l, const double* r,
                                    const double* omega, const double* ns_part, int order,
                                    const int32_t* factor_plan, int64_t plan_len,
                                    const double* consts, int64_t nconsts, int doubling_sum,
                                    int concurrent, void* const* input_ready_events,
                                    void* const* output_done_events, double* g_out,
                                    double* f_out, double* l_out, double* r_out,
                                    double* omega_out, double* ns_out, double* theta_out,
                                    int64_t* counters, void* stream) {
  return recursive_step_impl(h, n, nrhs, a, b, theta, g, f, l, r, omega, ns_part, order,
                             factor_plan, plan_len, consts, nconsts, doubling_sum, concurrent,
                             input_ready_events, output_done_events, g_out, f_out, l_out, r_out,
                             omega_out, ns_out, theta_out, counters, stream);
}

int si_plain_richardson(si_handle h, int64_t n, int64_t nrhs, const double* a, const double* b,
                        const double* theta, const double* p, double* theta_out,
                        int64_t* counters, void* stream) {
  return guard([&] {
    need(h && a && b && theta && p && theta_out, "null pointer");
    need(nrhs >= 1, "nrhs must be >= 1");
    Call call(h, stream, counters);
    plain_richardson(call.c, sq(a, n), rect(b, n, nrhs), rect(theta, n, nrhs), sq(p, n),
                     rect(theta_out, n, nrhs));
  });
}

// ---------------- block-row sharded steps ----------------

int si_comm_unique_id(unsigned char id[128]) {
  return guard([&] {
    need(id != nullptr, "null pointer");
    if (!nccl_unique_id(id)) throw Error(kECuda, "ncclGetUniqueId failed (is libnccl.so.2 present?)");
  });
}

int si_comm_create_nccl(si_handle h, int nranks, int rank, const unsigned char id[128], int64_t n,
                        si_comm* out) {
  return guard([&] {
    need(h && id && out, "null pointer");
    need(nranks >= 1 && rank >= 0 && rank < nranks && n >= nranks, "bad communicator shape");
    check(cudaSetDevice(h->h.device), "cudaSetDevice");
    auto c = std::make_unique<si_comm_s>();
    c->ex = make_nccl_exchange(nranks, rank, id);
    c->rank = rank;
    c->world = nranks;
    c->n = n;
    *out = c.release();
  });
}

int si_comm_create_callback(int nranks, int rank, int64_t n, si_allgather_fn allgather,
                            si_allreduce_fn allreduce, void* ctx, si_comm* out) {
  return guard([&] {
    need(allgather && allreduce && out, "null pointer");
    need(nranks >= 1 && rank >= 0 && rank < nranks && n >= nranks, "bad communicator shape");
    auto c = std::make_unique<si_comm_s>();
    c->ex = make_callback_exchange(allgather, allreduce, ctx);
    c->rank = rank;
    c->world = nranks;
    c->n = n;
    *out = c.release();
  });
}

int si_comm_destroy(si_comm c) {
  return guard([&] { delete c; });
}

int si_comm_rows(si_comm c, int64_t* r0, int64_t* r1, int64_t* gathers, int64_t* bytes_in) {
  return guard([&] {
    need(c != nullptr, "null communicator");
    Shard sh;
    sh.init(c->n, c->rank, c->world);
    if (r0) *r0 = sh.r0;
    if (r1) *r1 = sh.r1;
    if (gathers) *gathers = c->gathers;
    if (bytes_in) *bytes_in = c->bytes_in;
  });
}

int si_sharded_ns_step(si_handle h, si_comm comm, int64_t n, const double* a, const double* g_rows,
                       const double* f_rows, int order, const int32_t* plan, int64_t plan_len,
                       const double* consts, int64_t nconsts, double* g_out_rows,
                       double* f_out_rows, int64_t* counters, void* stream) {
  return guard([&] {
    need(h && a && g_rows && f_rows && g_out_rows && f_out_rows, "null pointer");
    PlanPtr pl = opt_plan(plan, plan_len, consts, nconsts);
    ShardCall sc(h, comm, n, stream, counters);
    mark_stable(sc.call.c, n, {a}, {g_out_rows, f_out_rows}, sc.rows());
    ns_step(sc.call.c, sq(a, n), sc.loc(g_rows, n), sc.loc(f_rows, n), order, pl.get(),
            sc.loc(g_out_rows, n), sc.loc(f_out_rows, n));
  });
}

int si_sharded_composite_step(si_handle h, si_comm comm, int64_t n, const double* a,
                              const double* g_rows, const double* f_rows, const double* precond,
                              const double* residual, const double* split_matrix, int nrates,
                              const int32_t* rates, const int32_t* plans,
                              const int64_t* plan_offsets, const double* consts, int64_t nconsts,
                              int order_n, double* g_out_rows, double* f_out_rows,
                              int64_t* counters, void* stream) {
  return guard([&] {
    need(h && a && g_rows && f_rows && precond && residual && split_matrix && g_out_rows &&
             f_out_rows,
         "null pointer");
    need(nrates >= 1 && rates, "composite spec needs at least one rate");
    need(order_n >= 1, "order_n must be >= 1");
    std::vector<int> rv(rates, rates + nrates);
    std::vector<PlanPtr> owned(nrates);
    std::vector<const PlanNode*> pv(nrates, nullptr);
    for (int i = 0; i < nrates; ++i) {
      need(rv[i] >= 1, "rates must be positive integers");
      if (plans && plan_offsets && plan_offsets[i + 1] > plan_offsets[i]) {
        owned[i] = decode_plan(plans + plan_offsets[i], plan_offsets[i + 1] - plan_offsets[i],
                               consts, nconsts);
        pv[i] = owned[i].get();
      }
    }
    ShardCall sc(h, comm, n, stream, counters);
    // the replicated inputs (and their row blocks) may keep their operand images
    mark_stable(sc.call.c, n, {a, precond, residual, split_matrix}, {g_out_rows, f_out_rows},
                sc.rows());
    // serial order only: every rank must issue its exchanges in the same order
    composite_step(sc.call.c, sq(a, n), sc.loc(g_rows, n), sc.loc(f_rows, n), sq(precond, n),
                   sq(residual, n), sq(split_matrix, n), rv, pv, order_n, false,
                   sc.loc(g_out_rows, n), sc.loc(f_out_rows, n));
  });
}

int si_sharded_richardson_recursive_step(
    si_handle h, si_comm comm, int64_t n, int64_t nrhs, const double* a, const double* b,
    const double* theta, const double* g_rows, const double* f_rows, const double* l_rows,
    const double* r_rows, const double* omega_rows, const double* ns_rows, int order,
    const int32_t* factor_plan, int64_t plan_len, const double* consts, int64_t nconsts,
    int doubling_sum, double* g_out_rows, double* f_out_rows, double* l_out_rows,
    double* r_out_rows, double* omega_out_rows, double* ns_out_rows, double* theta_out,
    int64_t* counters, void* stream) {
  return guard([&] {
    need(h && a && b && theta && g_rows && f_rows && l_rows && r_rows && g_out_rows &&
             f_out_rows && l_out_rows && r_out_rows && omega_out_rows && ns_out_rows && theta_out,
         "null pointer");
    need(nrhs >= 1, "nrhs must be >= 1");
    need((omega_rows == nullptr) == (ns_rows == nullptr), "omega and ns_part go together");
    PlanPtr pl = opt_plan(factor_plan, plan_len, consts, nconsts);
    if (pl) need(plan_order_of(*pl) == order, "factor plan order != iteration order");
    ShardCall sc(h, comm, n, stream, counters);
    mark_stable(sc.call.c, n, {a}, {g_out_rows, f_out_rows, l_out_rows, r_out_rows},
                sc.rows());
    MV om = omega_rows ? sc.loc(omega_rows, n) : MV{};
    MV nsp = ns_rows ? sc.loc(ns_rows, n) : MV{};
    richardson_recursive_step(sc.call.c, sq(a, n), rect(b, n, nrhs), rect(theta, n, nrhs),
                              sc.loc(g_rows, n), sc.loc(f_rows, n), sc.loc(l_rows, n),
                              sc.loc(r_rows, n), omega_rows ? &om : nullptr,
                              ns_rows ? &nsp : nullptr, order, false, pl.get(), doubling_sum != 0,
                              sc.loc(g_out_rows, n), sc.loc(f_out_rows, n), sc.loc(l_out_rows, n),
                              sc.loc(r_out_rows, n), sc.loc(omega_out_rows, n),
                              sc.loc(ns_out_rows, n), rect(theta_out, n, nrhs));
  });
}

int si_sharded_plain_richardson(si_handle h, si_comm comm, int64_t n, int64_t nrhs,
                                const double* a, const double* b, const double* theta,
                                const double* p_rows, double* theta_out, int64_t* counters,
                                void* stream) {
  return guard([&] {
    need(h && a && b && theta && p_rows && theta_out, "null pointer");
    need(nrhs >= 1, "nrhs must be >= 1");
    ShardCall sc(h, comm, n, stream, counters);
    plain_richardson(sc.call.c, sq(a, n), rect(b, n, nrhs), rect(theta, n, nrhs),
                     sc.loc(p_rows, n), rect(theta_out, n, nrhs));
  });
}

int si_sharded_fro_norm(si_handle h, si_comm comm, int64_t n, int64_t cols, const double* x_rows,
                        double* out, void* stream) {
  return guard([&] {
    need(h && x_rows && out, "null pointer");
    ShardCall sc(h, comm, n, stream, nullptr);
    *out = shard_fro(sc.call.c, sc.loc(x_rows, cols));
  });
}

int si_profile_begin(si_handle h) {
  return guard([&] {
    need(h != nullptr, "null handle");
    std::lock_guard<std::recursive_mutex> lock(h->h.mu);
    Handle& hh = h->h;
    for (auto* v : {&hh.prof, &hh.prof_i8}) {
      for (auto& r : *v) {
        hh.prof_pool.push_back(r.start);
        hh.prof_pool.push_back(r.stop);
      }
      v->clear();
    }
    hh.launches = 0;
    hh.profiling = true;
  });
}

int si_profile_end(si_handle h, double* gemm_ms, double* gemm_flops, int64_t* gemm_launches,
                   int64_t* total_launches) {
  return guard([&] {
    need(h != nullptr, "null handle");
    std::lock_guard<std::recursive_mutex> lock(h->h.mu);
    Handle& hh = h->h;
    hh.profiling = false;
    double ms = 0.0, fl = 0.0;
    for (auto& r : hh.prof) {
      check(cudaEventSynchronize(r.stop), "cudaEventSynchronize");
      float t = 0.f;
      check(cudaEventElapsedTime(&t, r.start, r.stop), "cudaEventElapsedTime");
      ms += t;
      fl += r.flops;
    }
    if (gemm_ms) *gemm_ms = ms;
    if (gemm_flops) *gemm_flops = fl;
    if (gemm_launches) *gemm_launches = (int64_t)hh.prof.size();
    if (total_launches) *total_launches = hh.launches;
  });
}

int si_dmma_peak(si_handle h, int iters, double* tflops) {
  return guard([&] {
    need(h && tflops && iters > 0, "bad arguments");
    check(cudaSetDevice(h->h.device), "cudaSetDevice");
    check(dmma_peak_tflops(iters, tflops), "dmma peak");
  });
}

int si_batched_composite_richardson(si_handle h, int64_t batch, int64_t n, const double* a,
                                    const double* b, const double* precond,
                                    const double* residual, int nrates, const int32_t* rates,
                                    const int32_t* plans, const int64_t* plan_offsets,
                                    const double* consts, int64_t nconsts, int order_n,
                                    int iters, double* p_io, double* f_io, double* theta_io,
                                    int64_t* counters, void* stream) {
  return si_batched_composite_richardson_ex(h, batch, n, a, b, precond, residual, nrates, rates,
                                            plans, plan_offsets, consts, nconsts, order_n, iters,
                                            p_io, f_io, theta_io, p_io, f_io, theta_io, counters,
                                            stream);
}

int si_batched_composite_richardson_ex(si_handle h, int64_t batch, int64_t n, const double* a,
                                       const double* b, const double* precond,
                                       const double* residual, int nrates, const int32_t* rates,
                                       const int32_t* plans, const int64_t* plan_offsets,
                                       const double* consts, int64_t nconsts, int order_n,
                                       int iters, const double* p_in, const double* f_in,
                                       const double* theta_in, double* p_out, double* f_out,
                                       double* theta_out, int64_t* counters, void* stream) {
  return si_batched_composite_richardson_gated(
      h, batch, n, a, b, precond, residual, nrates, rates, plans, plan_offsets, consts, nconsts,
      order_n, iters, p_in, f_in, theta_in, p_out, f_out, theta_out, nullptr, 0, 1, nullptr,
      counters, stream);
}

int si_batched_composite_richardson_gated(
    si_handle h, int64_t batch, int64_t n, const double* a, const double* b, const double* precond,
    const double* residual, int nrates, const int32_t* rates, const int32_t* plans,
    const int64_t* plan_offsets, const double* consts, int64_t nconsts, int order_n, int iters,
    const double* p_in, const double* f_in, const double* theta_in, double* p_out, double* f_out,
    double* theta_out, const uint32_t* chunk_ready, uint32_t epoch, int64_t chunk,
    uint32_t* chunk_done, int64_t* counters, void* stream) {
  return guard([&] {
    need(!chunk_ready || chunk >= 1, "chunk must be >= 1");
    // done counters are bumped by the gated kernel only: without input flags
    // (or with no iteration to run) nothing would ever raise them and a copy
    // stream waiting on them (si_stream_wait_u32) would hang.
    need(!chunk_done || chunk_ready, "chunk_done needs chunk_ready");
    need(!chunk_ready || iters >= 1, "a gated call needs iters >= 1");
    need(h && a && b && precond && residual && rates && p_in && f_in && theta_in && p_out &&
             f_out && theta_out,
         "null pointer");
    need(batch >= 0 && n >= 1 && n <= kBatchMaxN, "batched path supports 1 <= n <= 64");
    need(nrates >= 1 && nrates <= kBatchMaxRates, "batched path supports 1..4 rates");
    need(order_n >= 1 && iters >= 0, "bad order_n / iters");
    std::vector<int> rv(rates, rates + nrates);
    std::vector<PlanPtr> owned(nrates);
    std::vector<const PlanNode*> pv(nrates, nullptr);
    for (int i = 0; i < nrates; ++i) {
      need(rv[i] >= 1, "rates must be positive integers");
      if (plans && plan_offsets && plan_offsets[i + 1] > plan_offsets[i]) {
        owned[i] = decode_plan(plans + plan_offsets[i], plan_offsets[i + 1] - plan_offsets[i],
                               consts, nconsts);
        pv[i] = owned[i].get();
      }
    }
    Call call(h, stream, nullptr);
    ChunkGate gate;
    gate.ready = chunk_ready;
    gate.done = chunk_done;
    gate.epoch = epoch;
    gate.chunk = chunk;
    Counters per = batched_composite_richardson(call.c, batch, n, a, b, precond, residual, rv, pv,
                                                order_n, iters, p_in, f_in, theta_in, p_out,
                                                f_out, theta_out, chunk_ready ? &gate : nullptr);
    if (counters) {
      counters[0] += per.mmm;
      counters[1] += per.mvm;
    }
  });
}

int si_resident_program_source(int64_t n, int nrates, const int32_t* rates, const int32_t* plans,
                               const int64_t* plan_offsets, const double* consts,
                               int64_t nconsts, int order_n, char* out, int64_t cap,
                               int64_t* len) {
  return guard([&] {
    need(rates && len && nrates >= 1 && nrates <= kBatchMaxRates && order_n >= 1, "bad arguments");
    std::vector<int> rv(rates, rates + nrates);
    std::vector<PlanPtr> owned(nrates);
    std::vector<const PlanNode*> pv(nrates, nullptr);
    for (int i = 0; i < nrates; ++i)
      if (plans && plan_offsets && plan_offsets[i + 1] > plan_offsets[i]) {
        owned[i] = decode_plan(plans + plan_offsets[i], plan_offsets[i + 1] - plan_offsets[i],
                               consts, nconsts);
        pv[i] = owned[i].get();
      }
    const std::string src = resident_program_source(n, rv, pv, order_n);
    *len = (int64_t)src.size();
    if (out && cap > (int64_t)src.size()) std::memcpy(out, src.c_str(), src.size() + 1);
  });
}

int si_resident_program_source_ns(int64_t n, int order, int cluster, char* out, int64_t cap,
                                  int64_t* len) {
  return guard([&] {
    need(len && order >= 1 && (cluster == 2 || cluster == 4 || cluster == 8), "bad arguments");
    const std::string src = resident_program_source_ns(n, order, cluster);
    *len = (int64_t)src.size();
    if (out && cap > (int64_t)src.size()) std::memcpy(out, src.c_str(), src.size() + 1);
  });
}

int si_batched_ns_richardson(si_handle h, int64_t batch, int64_t n, const double* a,
                             const double* b, int order, const int32_t* plan, int64_t plan_len,
                             const double* consts, int64_t nconsts, int iters, double* p_io,
                             double* f_io, double* theta_io, int64_t* counters, void* stream) {
  return si_batched_ns_richardson_ex(h, batch, n, a, b, order, plan, plan_len, consts, nconsts,
                                     iters, p_io, f_io, theta_io, p_io, f_io, theta_io, counters,
                                     stream);
}

int si_batched_ns_richardson_ex(si_handle h, int64_t batch, int64_t n, const double* a,
                                const double* b, int order, const int32_t* plan,
                                int64_t plan_len, const double* consts, int64_t nconsts,
                                int iters, const double* p_in, const double* f_in,
                                const double* theta_in, double* p_out, double* f_out,
                                double* theta_out, int64_t* counters, void* stream) {
  return guard([&] {
    need(h && a && b && p_in && f_in && theta_in && p_out && f_out && theta_out, "null pointer");
    need(batch >= 0 && n >= 1 && n <= kBatchMaxN, "batched path supports 1 <= n <= 64");
    need(order >= 1 && iters >= 0, "bad order / iters");
    PlanPtr pl = opt_plan(plan, plan_len, consts, nconsts);
    if (pl) need(plan_order_of(*pl) == order, "plan order != iteration order");
    Call call(h, stream, nullptr);
    Counters per = batched_ns_richardson(call.c, batch, n, a, b, order, pl.get(), iters, p_in,
                                         f_in, theta_in, p_out, f_out, theta_out);
    if (counters) {
      counters[0] += per.mmm;
      counters[1] += per.mvm;
    }
  });
}

}  // extern "C"

/* ---------------- FP64 product backend (ozaki.cu) ---------------- */

int si_set_gemm_backend(si_handle h, int backend, int nmoduli, int64_t min_dim) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(backend == SI_GEMM_DMMA || backend == SI_GEMM_OZAKI_I8, "unknown backend");
    need(nmoduli == 0 || (nmoduli >= oz::kMinModuli && nmoduli <= oz::kMaxModuli),
         "nmoduli out of range");
    need(min_dim >= 0, "negative min_dim");
    std::lock_guard<std::recursive_mutex> lock(h->h.mu);
    h->h.gemm_backend = backend;
    if (nmoduli) h->h.oz_nmod = nmoduli;
    if (min_dim) h->h.oz_min_dim = std::max<int64_t>(min_dim, 128);
  });
}

int si_get_gemm_backend(si_handle h, int* backend, int* nmoduli, int64_t* min_dim) {
  return guard([&] {
    need(h != nullptr, "null handle");
    std::lock_guard<std::recursive_mutex> lock(h->h.mu);
    if (backend) *backend = h->h.gemm_backend;
    if (nmoduli) *nmoduli = h->h.oz_nmod;
    if (min_dim) *min_dim = h->h.oz_min_dim;
  });
}

int si_set_ozaki_chunks(si_handle h, int64_t max_rows, int64_t max_cols) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(max_rows >= 0 && max_cols >= 0, "negative chunk bound");
    std::lock_guard<std::recursive_mutex> lock(h->h.mu);
    h->h.oz_max_rows = max_rows;
    h->h.oz_max_cols = max_cols;
  });
}

int si_set_ozaki_kernel(si_handle h, int variant) {
  return guard([&] {
    need(h != nullptr, "null handle");
    need(variant == oz::kI8Auto || variant == oz::kI8Pair || variant == oz::kI8Single ||
             variant == oz::kI8Multicast,
         "unknown INT8 kernel variant");
    std::lock_guard<std::recursive_mutex> lock(h->h.mu);
    h->h.oz_variant = variant;
  });
}

int si_ozaki_tune(int group_m, int l2_a, int l2_b) {
  return guard([&] {
    need(group_m >= 0 && l2_a >= -1 && l2_a <= 2 && l2_b >= -1 && l2_b <= 2, "bad tuning values");
    oz::tune_pair(group_m, l2_a, l2_b);
  });
}

int si_ozaki_tune_stages(int stages) {
  return guard([&] {
    need(stages >= 3 && stages <= 6, "stages out of range");
    oz::tune_pair_stages(stages);
  });
}

int si_ozaki_tune_ksplit(int64_t kmax) {
  return guard([&] {
    need(kmax >= 0 && kmax % 128 == 0, "kmax must be a non-negative multiple of 128");
    oz::tune_ksplit(kmax);
  });
}

int si_ozaki_moduli(int n, uint32_t* moduli) {
  return guard([&] {
    need(moduli != nullptr && n >= 1 && n <= oz::kMaxModuli, "bad arguments");
    for (int l = 0; l < n; ++l) moduli[l] = oz::modulus(l);
  });
}

int si_i8_gemm_mod(si_handle h, const int8_t* a, const int8_t* bt, uint8_t* r, int64_t m,
                   int64_t n, int64_t kp, int nplanes, void* stream) {
  return guard([&] {
    need(h && a && bt && r, "null pointer");
    need(m > 0 && n > 0 && kp > 0 && kp % 128 == 0, "bad shape (kp must be a multiple of 128)");
    need(kp <= oz::kMaxK, "kp too large");
    need(nplanes >= 1 && nplanes <= oz::kMaxModuli, "nplanes out of range");
    Call call(h, stream, nullptr);
    check(oz::launch_i8_gemm_mod(a, bt, r, m, n, kp, nplanes, call.c.s, h->h.oz_variant),
          "i8 gemm launch");
    h->h.launches += 1;
  });
}

int si_profile_i8(si_handle h, double* ms, double* ops, int64_t* launches) {
  return guard([&] {
    need(h != nullptr, "null handle");
    std::lock_guard<std::recursive_mutex> lock(h->h.mu);
    double t = 0.0, o = 0.0;
    for (auto& r : h->h.prof_i8) {
      check(cudaEventSynchronize(r.stop), "cudaEventSynchronize");
      float x = 0.f;
      check(cudaEventElapsedTime(&x, r.start, r.stop), "cudaEventElapsedTime");
      t += x;
      o += r.flops;
    }
    if (ms) *ms = t;
    if (ops) *ops = o;
    if (launches) *launches = (int64_t)h->h.prof_i8.size();
  });
}
