// Step bodies of newton_schulz.py and richardson.py on the native engine.
// Outputs are caller-owned device buffers; inputs are never written (the
// reference's purity contract: states are immutable, matrix_core.py:52).
#include <functional>
#include "steps.hpp"

namespace si {

// ns:127-147
void initial_series(Ctx& c, const MV& P, const MV& B, const MV& A, int p, int w, const MV& Gout,
                    const MV& Fout) {
  if (p < 0 || w < 1) throw Error(kEInval, "requires p >= 0 and w >= 1");
  const int h = w * (p + 1);
  if (h == 1) {
    copy_into(c, Gout, P);
    copy_into(c, Fout, B);
    return;
  }
  MV g = factored(c, B, P, A, p, w);
  copy_into(c, Gout, g);
  residual_into(c, Fout, Gout, A);
}

// F' = I - G' A in `chunks` row blocks, events[k] recorded after block k (its
// rows may go device->host while the next block is computed); one counted
// product, as in the reference DAG.
static void residual_chunked(Ctx& c, const MV& Fout, const MV& Gout, const MV& A, int chunks,
                             const cudaEvent_t* events) {
  const int64_t n = Fout.v.rows;
  for (int k = 0; k < chunks; ++k) {
    const int64_t r0 = n * k / chunks, r1 = n * (k + 1) / chunks;
    MV fr = view(Fout.v.p + r0 * Fout.v.ld, r1 - r0, Fout.v.cols, Fout.v.ld);
    MV gr = view(Gout.v.p + r0 * Gout.v.ld, r1 - r0, Gout.v.cols, Gout.v.ld);
    gemm(c, fr, gr, A, -1.0, nullptr, 0.0, 1.0, false, r0);  // rows of I - G'A
    if (events && events[k]) check(cudaEventRecord(events[k], c.s), "cudaEventRecord");
  }
  c.ctr.mmm -= chunks - 1;
}

// ns:150-174
void ns_step(Ctx& c, const MV& A, const MV& G, const MV& F, int order, const PlanNode* plan,
             const MV& Gout, const MV& Fout, cudaEvent_t g_done, int f_chunks,
             const cudaEvent_t* f_chunk) {
  if (order < 1) throw Error(kEInval, "order must be >= 1");
  MV g;
  if (plan) {
    if (plan_order_of(*plan) != order) throw Error(kEInval, "plan order != iteration order");
    g = eval_node(c, *plan, F, G, A);
  } else {
    g = horner(c, F, G, order);
  }
  copy_into(c, Gout, g);
  if (g_done) check(cudaEventRecord(g_done, c.s), "cudaEventRecord");  // G' may go D2H now
  if (f_chunks > 0)
    residual_chunked(c, Fout, Gout, A, f_chunks, f_chunk);
  else
    residual_into(c, Fout, Gout, A);
}

// ns:177-228 -- parts (T_i, Gamma_i) are independent of each other and of the
// state; with `concurrent` each part (and the NS part) runs on its own stream.
void StepEvents::wait(Ctx& c, int i) {
  if (i >= 0 && i < kInputs && ready[i] && !waited[i]) {
    check(cudaStreamWaitEvent(c.s, ready[i], 0), "cudaStreamWaitEvent");
    waited[i] = true;
  }
}

void composite_step(Ctx& c, const MV& A, const MV& G, const MV& F, const MV& P, const MV& B,
                    const MV& Sm, const std::vector<int>& rates,
                    const std::vector<const PlanNode*>& plans, int order_n, bool concurrent,
                    const MV& Gout, const MV& Fout, StepEvents* ev) {
  if (order_n < 1) throw Error(kEInval, "order_n must be >= 1");
  if (rates.empty()) throw Error(kEInval, "composite spec needs at least one rate");
  const size_t k = rates.size();
  std::vector<MV> ts(k), gs(k);
  MV nsp;
  StepEvents none;
  StepEvents& e = ev ? *ev : none;
  if (concurrent)  // branches read every input: wait for all of them up front
    for (int i = 0; i < StepEvents::kInputs; ++i) e.wait(c, i);
  // serial order of first use: S^-1, B, split matrix (parts), A (their
  // residuals), then G, F (the NS part) -- copies still in flight for the later
  // inputs overlap the first products
  e.wait(c, StepEvents::kPrecond);
  e.wait(c, StepEvents::kResidual);
  e.wait(c, StepEvents::kSplitMatrix);
  auto series = [&](Ctx& cc, size_t i) {  // T_i: products with B and S^-1 only
    if (rates[i] < 1) throw Error(kEInval, "rates must be positive integers");
    if (rates[i] == 1) {
      ts[i] = alloc_like(cc, P);
      copy_into(cc, ts[i], P);
    } else {
      ts[i] = geometric(cc, B, P, rates[i], Sm, plans[i]);
    }
  };
  auto part = [&](Ctx& cc, size_t i) {
    series(cc, i);
    e.wait(cc, StepEvents::kA);
    gs[i] = residual(cc, ts[i], A);
  };
  if (concurrent) {
    Fork fk(c);
    std::vector<Ctx> kids;
    const int nstreams = Handle::kSide - 1;
    for (int s = 0; s < nstreams && s < (int)k; ++s) kids.push_back(fk.branch(s));
    for (size_t i = 0; i < k; ++i) part(kids[i % kids.size()], i);
    Ctx nsc = fk.branch(Handle::kSide - 1);
    nsp = horner(nsc, F, G, order_n);
    for (auto& kd : kids) fk.join(kd);
    fk.join(nsc);
  } else {
    // every part's series first (they read only B and S^-1), then the
    // residuals Gamma_i = I - T_i A: with A still in flight (the e2e path)
    // its copy overlaps ten products instead of stalling the second; the
    // products are the same, so the results are bitwise unchanged
    for (size_t i = 0; i < k; ++i) series(c, i);
    e.wait(c, StepEvents::kA);
    for (size_t i = 0; i < k; ++i) gs[i] = residual(c, ts[i], A);
  }
  MV t = ts[0], r = gs[0];
  for (size_t i = 1; i < k; ++i) {
    t = gemm_new(c, r, ts[i], 1.0, &t, 1.0);  // t + r T_i
    r = gemm_new(c, r, gs[i]);                // r Gamma_i
  }
  if (!concurrent) {
    e.wait(c, StepEvents::kF);
    e.wait(c, StepEvents::kG);
    nsp = horner(c, F, G, order_n);
  }
  if (e.f_chunks > 0 && e.f_chunk && !c.shard) {
    // G' = t + r ns and F' = I - G' A in row blocks, interleaved: block k of
    // both is final at event k, so both go device->host while the next block
    // is computed (ns's operand image is built once: a stable value); two
    // counted products, as in the reference DAG
    keep_stable(c, nsp);
    const int64_t n = Gout.v.rows;
    const int chunks = e.f_chunks;
    auto rows = [](const MV& m, int64_t r0, int64_t r1) {
      return view(m.v.p + r0 * m.v.ld, r1 - r0, m.v.cols, m.v.ld);
    };
    for (int k = 0; k < chunks; ++k) {
      const int64_t r0 = n * k / chunks, r1 = n * (k + 1) / chunks;
      const MV gr = rows(Gout, r0, r1), tr = rows(t, r0, r1);
      gemm(c, gr, rows(r, r0, r1), nsp, 1.0, &tr, 1.0);          // rows of t + r ns
      if (k == chunks - 1 && e.g_done) check(cudaEventRecord(e.g_done, c.s), "cudaEventRecord");
      gemm(c, rows(Fout, r0, r1), gr, A, -1.0, nullptr, 0.0, 1.0, false, r0);  // rows of I - G'A
      if (e.f_chunk[k]) check(cudaEventRecord(e.f_chunk[k], c.s), "cudaEventRecord");
    }
    c.ctr.mmm -= 2 * (chunks - 1);
    return;
  }
  gemm(c, Gout, r, nsp, 1.0, &t, 1.0);  // G = t + r ns
  if (e.g_done) check(cudaEventRecord(e.g_done, c.s), "cudaEventRecord");  // G' may go D2H now
  if (e.f_chunks > 0 && e.f_chunk) {
    residual_chunked(c, Fout, Gout, A, e.f_chunks, e.f_chunk);
    return;
  }
  residual_into(c, Fout, Gout, A);
}

// Opt-in hoisting (not in the reference, which recomputes them every step):
// the state-independent half of composite_step (ns:204-216), T_comp and R_comp.
void composite_parts(Ctx& c, const MV& A, const MV& P, const MV& B, const MV& Sm,
                     const std::vector<int>& rates, const std::vector<const PlanNode*>& plans,
                     const MV& Tout, const MV& Rout) {
  if (rates.empty()) throw Error(kEInval, "composite spec needs at least one rate");
  MV t, r;
  for (size_t i = 0; i < rates.size(); ++i) {
    if (rates[i] < 1) throw Error(kEInval, "rates must be positive integers");
    MV ti;
    if (rates[i] == 1) {
      ti = alloc_like(c, P);
      copy_into(c, ti, P);
    } else {
      ti = geometric(c, B, P, rates[i], Sm, plans[i]);
    }
    MV gi = residual(c, ti, A);
    if (i == 0) {
      t = ti;
      r = gi;
    } else {
      t = gemm_new(c, r, ti, 1.0, &t, 1.0);
      r = gemm_new(c, r, gi);
    }
  }
  copy_into(c, Tout, t);
  copy_into(c, Rout, r);
}

// The state-dependent half (ns:218-220) with hoisted T_comp / R_comp.
void composite_apply(Ctx& c, const MV& A, const MV& G, const MV& F, const MV& T, const MV& R,
                     int order_n, const MV& Gout, const MV& Fout) {
  if (order_n < 1) throw Error(kEInval, "order_n must be >= 1");
  MV nsp = horner(c, F, G, order_n);
  gemm(c, Gout, R, nsp, 1.0, &T, 1.0);
  residual_into(c, Fout, Gout, A);
}

// ns:231-251
void initial_double(Ctx& c, const MV& P, const MV& B, const MV& A, int p, int w, int order,
                    const MV& Gout, const MV& Fout, const MV& Lout, const MV& Rout) {
  initial_series(c, P, B, A, p, w, Gout, Fout);
  MV l0 = horner(c, Fout, Gout, order);
  copy_into(c, Lout, l0);
  residual_into(c, Rout, Lout, A);
}

// ns:254-298
void double_ns_step(Ctx& c, const MV& A, const MV& G, const MV& F, const MV& L, const MV& R,
                    int order, bool concurrent, const MV& Gout, const MV& Fout, const MV& Lout,
                    const MV& Rout) {
  if (order < 1) throw Error(kEInval, "order must be >= 1");
  MV nsp;
  auto accel = [&](Ctx& cc) {
    MV gamma = residual(cc, L, A);
    MV l = horner(cc, gamma, L, order);
    copy_into(cc, Lout, l);
    residual_into(cc, Rout, Lout, A);
  };
  if (concurrent) {
    Fork fk(c);
    Ctx c1 = fk.branch(0), c2 = fk.branch(1);
    accel(c1);
    nsp = horner(c2, F, G, order);
    fk.join(c1);
    fk.join(c2);
  } else {
    accel(c);
    nsp = horner(c, F, G, order);
  }
  gemm(c, Gout, Rout, nsp, 1.0, &Lout, 1.0);  // L' + R' ns
  residual_into(c, Fout, Gout, A);
}

// ns:301-325
void additive_correction_step(Ctx& c, const MV& A, const MV& Z, const MV& G, int p,
                              const MV& Zout, const MV& Gout) {
  if (p < 2) throw Error(kEInval, "order p must be >= 2");
  MV lprev = residual(c, Z, A);
  MV zn = horner(c, lprev, Z, p);
  copy_into(c, Zout, zn);
  MV fprev = residual(c, G, A);
  gemm(c, Gout, fprev, Zout, 1.0, &G, 1.0);
}

// ri:81-98
void richardson_step(Ctx& c, const MV& A, const MV& b, const MV& theta, const MV& G, const MV& F,
                     const MV& L, const MV& R, int order, int q, const MV& Gout, const MV& Fout,
                     const MV& Lout, const MV& Rout, const MV& theta_out) {
  if (q < 1) throw Error(kEInval, "q must be >= 1");
  double_ns_step(c, A, G, F, L, R, order, false, Gout, Fout, Lout, Rout);
  MV s = horner(c, Fout, Gout, q);
  MV wgt = gemm_new(c, Rout, s, 1.0, &Lout, 1.0);
  MV resid = gemm_new(c, A, theta, 1.0, &b, -1.0, 0.0, true);   // A theta - b
  gemm(c, theta_out, wgt, resid, -1.0, &theta, 1.0, 0.0, true);  // theta - W resid
}

// ri:101-108  I + gamma + ... + gamma^(n-1)
MV power_sum(Ctx& c, const MV& gamma, int n) {
  MV acc = identity_like(c, gamma);
  MV cur;
  bool have = false;
  for (int i = 0; i < n - 1; ++i) {
    cur = have ? gemm_new(c, cur, gamma) : gamma;
    have = true;
    acc = lincomb(c, 0.0, {{1.0, &acc}, {1.0, &cur}}, gamma.v.rows, gamma.v.cols);
  }
  return acc;
}

// Opt-in (not in the reference): S_n(gamma) for n = 2^m as the product of the
// factors (I + gamma^(2^j)), i.e. S_2t = S_t + gamma^t S_t: 2(m-1) products
// instead of the n-2 of power_sum.
MV power_sum_doubling(Ctx& c, const MV& gamma, int n) {
  if (n < 2 || (n & (n - 1))) throw Error(kEInval, "doubling power sum needs n = 2^m >= 2");
  MV eye = identity_like(c, gamma);
  MV s = lincomb(c, 0.0, {{1.0, &eye}, {1.0, &gamma}}, gamma.v.rows, gamma.v.cols);  // I + gamma
  MV pw = gamma;
  for (int t = 2; t < n; t *= 2) {
    pw = gemm_new(c, pw, pw);               // gamma^t
    s = gemm_new(c, pw, s, 1.0, &s, 1.0);   // S_2t = S_t + gamma^t S_t
  }
  return s;
}

// ri:111-189.  Opt-in factorised variant (not in the reference): `factor_plan`
// evaluates N' = S_n(F) G through a plan of order n and `doubling_sum` builds
// S_n(gamma) by power_sum_doubling (order 16: 18 products instead of 34).
void richardson_recursive_step(Ctx& c, const MV& A, const MV& b, const MV& theta, const MV& G,
                               const MV& F, const MV& L, const MV& R, const MV* omega,
                               const MV* ns_part, int order, bool concurrent,
                               const PlanNode* factor_plan, bool doubling_sum,
                               const MV& Gout, const MV& Fout, const MV& Lout, const MV& Rout,
                               const MV& omega_out, const MV& ns_out, const MV& theta_out,
                               const cudaEvent_t* out_done) {
  const int n = order;
  if (n < 1) throw Error(kEInval, "order must be >= 1");
  // an output may go device->host as soon as it is final (its event fires on
  // the stream that wrote it; later products only read it)
  auto done = [&](Ctx& cc, int which) {
    if (out_done && out_done[which])
      check(cudaEventRecord(out_done[which], cc.s), "cudaEventRecord");
  };
  MV ns_prev, om_prev;
  if (!omega || !ns_part) {
    ns_prev = horner(c, F, G, n);
    om_prev = gemm_new(c, R, ns_prev, 1.0, &L, 1.0);
  } else {
    ns_prev = *ns_part;
    om_prev = *omega;
  }
  MV s = doubling_sum ? power_sum_doubling(c, R, n) : power_sum(c, R, n);
  MV nsn;
  auto estimate_then = [&](Ctx& cc, const std::function<void(Ctx&)>& after_g) {
    {
      MV diff = lincomb(cc, 0.0, {{1.0, &om_prev}, {-1.0, &ns_prev}}, G.v.rows, G.v.cols);
      gemm(cc, Gout, s, diff, 1.0, &ns_prev, 1.0);  // S (om - ns) + ns
    }
    done(cc, kRecG);
    if (after_g) after_g(cc);
    residual_into(cc, Fout, Gout, A);
    done(cc, kRecF);
    nsn = factor_plan ? eval_node(cc, *factor_plan, Fout, Gout, A) : horner(cc, Fout, Gout, n);
  };
  auto estimate = [&](Ctx& cc) { estimate_then(cc, nullptr); };
  auto accel = [&](Ctx& cc) {
    gemm(cc, Lout, s, L);
    done(cc, kRecL);
    residual_into(cc, Rout, Lout, A);
    done(cc, kRecR);
  };
  if (concurrent) {
    Fork fk(c);
    Ctx c1 = fk.branch(0), c2 = fk.branch(1);
    estimate(c1);
    accel(c2);
    fk.join(c1);
    fk.join(c2);
  } else {
    // the independent accel half first: S is then last read by G' = S (om - ns)
    // + ns and released before F' and N' are formed (one n x n matrix less at
    // the step's peak; the emulated products' workspace needs it at n = 32768)
    accel(c);
    auto release_s = [&](Ctx&) {
      s = MV();
      ns_prev = MV();
      om_prev = MV();
    };
    estimate_then(c, release_s);
  }
  copy_into(c, ns_out, nsn);
  done(c, kRecNs);
  gemm(c, omega_out, Rout, ns_out, 1.0, &Lout, 1.0);              // L' + R' N'
  done(c, kRecOmega);
  MV resid = gemm_new(c, A, theta, 1.0, &b, -1.0, 0.0, true);     // A theta - b
  gemm(c, theta_out, omega_out, resid, -1.0, &theta, 1.0, 0.0, true);
  done(c, kRecTheta);
}

// theta + P (b - A theta), evaluated as ri:88-89 does.
void plain_richardson(Ctx& c, const MV& A, const MV& b, const MV& theta, const MV& P,
                      const MV& theta_out) {
  MV resid = gemm_new(c, A, theta, 1.0, &b, -1.0, 0.0, true);
  gemm(c, theta_out, P, resid, -1.0, &theta, 1.0, 0.0, true);
}

}  // namespace si
