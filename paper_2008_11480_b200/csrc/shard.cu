// Block-row sharded execution (see shard.hpp).
#include "shard.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

namespace si {

void Shard::init(int64_t n_, int rank_, int world_) {
  n = n_;
  rank = rank_;
  world = world_;
  // near-equal contiguous blocks, the first n % world one row longer
  // (sharded.py:row_splits)
  starts.assign(world + 1, 0);
  const int64_t base = n / world, extra = n % world;
  for (int p = 0; p < world; ++p) starts[p + 1] = starts[p] + base + (p < extra ? 1 : 0);
  r0 = starts[rank];
  r1 = starts[rank + 1];
  pad = base + (extra ? 1 : 0);
}

MV shard_rows(Ctx& c, const MV& x) {
  const Shard& sh = *c.shard;
  if (x.local) return x;
  if (x.v.rows != sh.n) throw Error(kEInval, "sharded call: operand is neither n rows nor local");
  MV r = view(x.v.p + sh.r0 * x.v.ld, sh.r1 - sh.r0, x.v.cols, x.v.ld);
  r.own = x.own;
  r.local = true;
  return r;
}

namespace {

// rows [0, rows) of a padded rank-major gather buffer block q -> D rows
void compact(Ctx& c, const MV& D, const double* recv, int64_t cols, int skip_rank) {
  const Shard& sh = *c.shard;
  for (int q = 0; q < sh.world; ++q) {
    if (q == skip_rank) continue;
    const int64_t rows = sh.starts[q + 1] - sh.starts[q];
    if (rows == 0) continue;
    Mat dst{D.v.p + sh.starts[q] * D.v.ld, rows, cols, D.v.ld};
    Mat src{const_cast<double*>(recv) + q * sh.pad * cols, rows, cols, cols};
    check(launch_copy(dst, src, c.s), "gather copy");
    c.h->launches += 1;
  }
}

// all-gather the local rows `loc` (rows r1 - r0, any ld) into D (n rows)
void gather(Ctx& c, const MV& loc, const MV& D, bool local_already_in_d) {
  Shard& sh = *c.shard;
  const int64_t cols = loc.v.cols, rows = sh.r1 - sh.r0;
  const bool even = sh.n == sh.pad * sh.world;
  sh.gathers += 1;
  sh.bytes_in += (sh.n - rows) * cols * 8;
  if (even && D.v.ld == cols) {
    // straight into D; NCCL's in-place form when the local rows are already there
    double* slot = D.v.p + sh.r0 * cols;
    if (!(local_already_in_d && loc.v.p == slot && loc.v.ld == cols)) {
      Mat dst{slot, rows, cols, cols};
      check(launch_copy(dst, loc.v, c.s), "gather copy");
      c.h->launches += 1;
    }
    sh.ex->allgather(slot, D.v.p, rows * cols, c.s);
    return;
  }
  MV send = alloc(c, sh.pad, cols);
  MV recv = alloc(c, sh.pad * sh.world, cols);
  {
    Mat dst{send.v.p, rows, cols, cols};
    check(launch_copy(dst, loc.v, c.s), "gather copy");
    c.h->launches += 1;
  }
  sh.ex->allgather(send.v.p, recv.v.p, sh.pad * cols, c.s);
  compact(c, D, recv.v.p, cols, local_already_in_d ? sh.rank : -1);
}

}  // namespace

MV shard_full(Ctx& c, const MV& x) {
  Shard& sh = *c.shard;
  if (!x.local) return x;
  for (auto it = sh.cache.begin(); it != sh.cache.end();) {
    const bool owned = it->key == nullptr;
    if (owned && it->src.expired()) {  // its source was freed: the address may be reused
      it = sh.cache.erase(it);
      continue;
    }
    const bool same = owned ? (x.own && it->src.lock() == x.own && it->full.v.cols == x.v.cols)
                            : (!x.own && it->key == x.v.p && it->full.v.cols == x.v.cols);
    if (same) return it->full;
    ++it;
  }
  MV full = alloc(c, sh.n, x.v.cols);
  gather(c, x, full, false);
  // owned values are matched by their storage, caller-owned inputs (no `own`)
  // by address: both are immutable for the duration of the call
  sh.cache.push_back({x.own, x.own ? nullptr : x.v.p, full});
  if (sh.cache.size() > 8) sh.cache.erase(sh.cache.begin());
  return full;
}

void shard_gather_into(Ctx& c, const MV& D) {
  MV loc = shard_rows(c, D);
  gather(c, loc, D, true);
}

double shard_fro(Ctx& c, const MV& x) {
  Shard& sh = *c.shard;
  MV loc = shard_rows(c, x);
  MV red = alloc(c, 1, (int64_t)reduce_work_elems(loc.v) + 1);
  double* out = red.v.p + reduce_work_elems(loc.v);
  check(launch_sumsq(loc.v, out, red.v.p, c.s), "sumsq");
  sh.ex->allreduce_sum(out, 1, c.s);
  double v = 0.0;
  check(cudaMemcpyAsync(&v, out, sizeof(double), cudaMemcpyDeviceToHost, c.s), "memcpy");
  check(cudaStreamSynchronize(c.s), "sync");
  return std::sqrt(v);
}

// ---------------------------------------------------------------------------
// NCCL through dlopen
// ---------------------------------------------------------------------------

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allgather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*err)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer a libnccl already in the process (e.g. PyTorch's), then the system one
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return;
    auto sym = [&](const char* name) { return dlsym(lib, name); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(sym("ncclCommInitRank"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(sym("ncclCommDestroy"));
    api.allgather = reinterpret_cast<decltype(api.allgather)>(sym("ncclAllGather"));
    api.allreduce = reinterpret_cast<decltype(api.allreduce)>(sym("ncclAllReduce"));
    api.err = reinterpret_cast<decltype(api.err)>(sym("ncclGetErrorString"));
    api.ok = api.get_unique_id && api.init_rank && api.destroy && api.allgather &&
             api.allreduce && api.err;
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  throw Error(kECuda, std::string(what) + ": " + nccl().err(r));
}

struct NcclExchange : Exchange {
  ncclComm_t comm = nullptr;
  ~NcclExchange() override {
    if (comm) nccl().destroy(comm);
  }
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t s) override {
    nccl_check(nccl().allgather(send, recv, (size_t)count, ncclDouble, comm, s), "ncclAllGather");
  }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t s) override {
    nccl_check(nccl().allreduce(buf, buf, (size_t)count, ncclDouble, ncclSum, comm, s),
               "ncclAllReduce");
  }
  const char* kind() const override { return "nccl"; }
};

struct CallbackExchange : Exchange {
  AllgatherFn ag;
  AllreduceFn ar;
  void* ctx;
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t s) override {
    if (ag(ctx, send, recv, count, s) != 0) throw Error(kECuda, "all-gather callback failed");
  }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t s) override {
    if (ar(ctx, buf, count, s) != 0) throw Error(kECuda, "all-reduce callback failed");
  }
  const char* kind() const override { return "callback"; }
};

}  // namespace

bool nccl_unique_id(unsigned char id[128]) {
  if (!nccl().ok) return false;
  ncclUniqueId u;
  if (nccl().get_unique_id(&u) != ncclSuccess) return false;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return true;
}

std::unique_ptr<Exchange> make_nccl_exchange(int nranks, int rank, const unsigned char id[128]) {
  if (!nccl().ok) throw Error(kECuda, "libnccl.so.2 could not be loaded");
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  auto ex = std::make_unique<NcclExchange>();
  nccl_check(nccl().init_rank(&ex->comm, nranks, u, rank), "ncclCommInitRank");
  return ex;
}

std::unique_ptr<Exchange> make_callback_exchange(AllgatherFn ag, AllreduceFn ar, void* ctx) {
  auto ex = std::make_unique<CallbackExchange>();
  ex->ag = ag;
  ex->ar = ar;
  ex->ctx = ctx;
  return ex;
}

}  // namespace si
