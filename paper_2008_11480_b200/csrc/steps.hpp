#pragma once
#include <vector>

#include "engine.hpp"

namespace si {

void initial_series(Ctx& c, const MV& P, const MV& B, const MV& A, int p, int w, const MV& Gout,
                    const MV& Fout);
// g_done (optional) is recorded once G' is final, before F' = I - G' A.
// Inputs in flight are registered on the Ctx (Ctx::awaits).
// f_chunks > 0: F' in that many row blocks, f_chunk[k] recorded after block k.
void ns_step(Ctx& c, const MV& A, const MV& G, const MV& F, int order, const PlanNode* plan,
             const MV& Gout, const MV& Fout, cudaEvent_t g_done = nullptr, int f_chunks = 0,
             const cudaEvent_t* f_chunk = nullptr);
// Optional per-input readiness (e.g. host->device copies still in flight on a
// copy stream): the step waits on each event just before the input's first
// use, and records g_done once G' is final (before F' = I - G' A).
struct StepEvents {
  enum { kA = 0, kG, kF, kPrecond, kResidual, kSplitMatrix, kInputs };
  cudaEvent_t ready[kInputs] = {};
  bool waited[kInputs] = {};
  cudaEvent_t g_done = nullptr;
  // F' = I - G' A in f_chunks row blocks, f_chunk[k] recorded after block k
  // (its rows may go device->host while the next block is computed)
  const cudaEvent_t* f_chunk = nullptr;
  int f_chunks = 0;
  void wait(Ctx& c, int i);
};
void composite_step(Ctx& c, const MV& A, const MV& G, const MV& F, const MV& P, const MV& B,
                    const MV& Sm, const std::vector<int>& rates,
                    const std::vector<const PlanNode*>& plans, int order_n, bool concurrent,
                    const MV& Gout, const MV& Fout, StepEvents* ev = nullptr);
void composite_parts(Ctx& c, const MV& A, const MV& P, const MV& B, const MV& Sm,
                     const std::vector<int>& rates, const std::vector<const PlanNode*>& plans,
                     const MV& Tout, const MV& Rout);
void composite_apply(Ctx& c, const MV& A, const MV& G, const MV& F, const MV& T, const MV& R,
                     int order_n, const MV& Gout, const MV& Fout);
void initial_double(Ctx& c, const MV& P, const MV& B, const MV& A, int p, int w, int order,
                    const MV& Gout, const MV& Fout, const MV& Lout, const MV& Rout);
void double_ns_step(Ctx& c, const MV& A, const MV& G, const MV& F, const MV& L, const MV& R,
                    int order, bool concurrent, const MV& Gout, const MV& Fout, const MV& Lout,
                    const MV& Rout);
void additive_correction_step(Ctx& c, const MV& A, const MV& Z, const MV& G, int p,
                              const MV& Zout, const MV& Gout);
void richardson_step(Ctx& c, const MV& A, const MV& b, const MV& theta, const MV& G, const MV& F,
                     const MV& L, const MV& R, int order, int q, const MV& Gout, const MV& Fout,
                     const MV& Lout, const MV& Rout, const MV& theta_out);
MV power_sum(Ctx& c, const MV& gamma, int n);
MV power_sum_doubling(Ctx& c, const MV& gamma, int n);
void richardson_recursive_step(Ctx& c, const MV& A, const MV& b, const MV& theta, const MV& G,
                               const MV& F, const MV& L, const MV& R, const MV* omega,
                               const MV* ns_part, int order, bool concurrent,
                               const PlanNode* factor_plan, bool doubling_sum,
                               const MV& Gout, const MV& Fout, const MV& Lout, const MV& Rout,
                               const MV& omega_out, const MV& ns_out, const MV& theta_out,
                               const cudaEvent_t* out_done = nullptr);
// indices of `out_done` (each may be null): recorded once that output is final
enum { kRecL = 0, kRecR, kRecG, kRecF, kRecNs, kRecOmega, kRecTheta, kRecOutputs };
void plain_richardson(Ctx& c, const MV& A, const MV& b, const MV& theta, const MV& P,
                      const MV& theta_out);

}  // namespace si
