// Block-row sharded execution of the step engine behind the
// C ABI (si_comm_* / si_sharded_*): every state matrix is split into
// contiguous row blocks, one per rank, A and the splitting are replicated.
// The engine's primitives (engine.cu) see Ctx::shard and
//   * compute only this rank's rows of every product (a replicated left or
//     epilogue operand is read through its row view, diag*I shifted to the
//     block's global diagonal),
//   * all-gather a sharded right operand before the product (once per value),
// so the step bodies of steps.cu run unchanged and execute the reference's
// GEMM DAG (same products, same counters, same per-tile K order: results are
// bitwise independent of the number of ranks).
#pragma once
#include <memory>
#include <vector>

#include "engine.hpp"

namespace si {

// The exchange of one communicator: all-gather of equal-size blocks
// (rank-major into recv) and an in-place sum, both stream-ordered.
struct Exchange {
  virtual ~Exchange() = default;
  virtual void allgather(const double* send, double* recv, int64_t count, cudaStream_t s) = 0;
  virtual void allreduce_sum(double* buf, int64_t count, cudaStream_t s) = 0;
  virtual const char* kind() const = 0;
};

// NCCL (loaded with dlopen when the first communicator is created, so the
// library itself has no link-time NCCL dependency).
bool nccl_unique_id(unsigned char id[128]);
std::unique_ptr<Exchange> make_nccl_exchange(int nranks, int rank, const unsigned char id[128]);

// Caller-provided exchange (e.g. a host transport in tests, or an MPI layer):
// both callbacks are called with the stream they must be ordered on.
using AllgatherFn = int (*)(void* ctx, const double* send, double* recv, int64_t count,
                            void* stream);
using AllreduceFn = int (*)(void* ctx, double* buf, int64_t count, void* stream);
std::unique_ptr<Exchange> make_callback_exchange(AllgatherFn ag, AllreduceFn ar, void* ctx);

struct Shard {
  Exchange* ex = nullptr;
  int rank = 0, world = 1;
  int64_t n = 0, r0 = 0, r1 = 0, pad = 0;
  std::vector<int64_t> starts;  // world + 1 row-block bounds
  // gathered copies of sharded values used as right operands in this call,
  // keyed by their storage (a value is immutable once produced)
  struct Entry {
    std::weak_ptr<Buf> src;
    const double* key;
    MV full;
  };
  std::vector<Entry> cache;
  int64_t gathers = 0;
  int64_t bytes_in = 0;  // bytes received from the other ranks
  void init(int64_t n_, int rank_, int world_);
};

MV shard_rows(Ctx& c, const MV& x);        // this rank's rows (x itself if already local)
MV shard_full(Ctx& c, const MV& x);        // the whole matrix (all-gather of a local value)
void shard_gather_into(Ctx& c, const MV& D);  // D replicated, its rows [r0, r1) computed: fill the rest
double shard_fro(Ctx& c, const MV& x);     // ||x||_F over all ranks (local sums + one all-reduce)

}  // namespace si
