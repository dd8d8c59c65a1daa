#pragma once
#include <string>
#include <vector>

#include "engine.hpp"

namespace si {

constexpr int kBatchMaxN = 64;

// Inputs arriving by chunks of `chunk` systems: chunk k's inputs are valid once
// ready[k] >= epoch (wrap-safe); done[k] (may be null) is incremented once per
// finished system of chunk k, after its outputs are written.
struct ChunkGate {
  const unsigned* ready = nullptr;
  unsigned* done = nullptr;
  unsigned epoch = 0;
  int64_t chunk = 1;
};
constexpr int kBatchMaxRates = 4;

// BASELINE config 2: `iters` x { plain Richardson with P_k;
// composite_step(rates, order_n) (newton_schulz.py:177-228) } for `batch`
// independent n x n systems, one CTA per system, state resident in shared
// memory across iterations.  Returns the per-system counter delta.
Counters batched_composite_richardson(Ctx& c, int64_t batch, int64_t n, const double* a,
                                      const double* b, const double* precond,
                                      const double* residual, const std::vector<int>& rates,
                                      const std::vector<const PlanNode*>& plans, int order_n,
                                      int iters, const double* p_in, const double* f_in,
                                      const double* theta_in, double* p_out, double* f_out,
                                      double* theta_out, const ChunkGate* gate = nullptr);

// BASELINE config 1 (batch = 1) and batches of it: `iters` x { plain
// Richardson with P_k; ns_step(order, plan) (newton_schulz.py:150-174) }.
Counters batched_ns_richardson(Ctx& c, int64_t batch, int64_t n, const double* a, const double* b,
                               int order, const PlanNode* plan, int iters, const double* p_in,
                               const double* f_in, const double* theta_in, double* p_out,
                               double* f_out, double* theta_out);
// Inputs may equal outputs (in place).

// The body of a compile-time program struct (FX of resident_kernel) for the
// composite recipe at n <= 32: the scheduled, slot-allocated op list and the
// bytes the launcher matches it against (tools/gen_resident_fixed.py).
std::string resident_program_source(int64_t n, const std::vector<int>& rates,
                                    const std::vector<const PlanNode*>& plans, int order_n);
// ... and for the NS recipe of config 1 (32 < n <= 64) in cluster mode with `cl` CTAs.
std::string resident_program_source_ns(int64_t n, int order, int cl);

}  // namespace si
