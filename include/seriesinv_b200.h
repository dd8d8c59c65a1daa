/*
 * seriesinv_b200.h -- C ABI of the B200-native seriesinv hot path.
 *
 * Drop-in boundary for the FP64 matrix-product chains of arXiv 2008.11480's
 * reference package `seriesinv` (/root/reference/pkg/src/seriesinv).  The
 * reference has no FFI of its own (pure Python + numpy); its seams are
 *   - the GEMM seam  mat_mul / mat_vec           (matrix_core.py:101-114), and
 *   - the step seam  ns_step, composite_step, ...  (newton_schulz.py:127-325,
 *                    richardson.py:61-189, series_toolkit.py:279-457).
 * Each entry point below names the reference function it replaces.
 *
 * Conventions
 *   - All matrix/vector pointers are DEVICE pointers to FP64 row-major data.
 *     Step-level functions take contiguous n x n matrices (ld = n) and
 *     contiguous n x nrhs right-hand sides (nrhs = 1 for a vector).
 *   - Output buffers are caller-owned and must not alias inputs; inputs are
 *     never written (the reference's states are immutable, matrix_core.py:52).
 *     Temporaries come from a handle-owned stream-ordered memory pool.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     asynchronous unless documented otherwise.
 *   - `counters` (may be NULL) points at int64_t[2] = {mmm, mvm}; each call ADDS
 *     the number of matrix-matrix / matrix-vector products it executed, which
 *     equals the reference MulCounter delta for the same call
 *     (matrix_core.py:71-98).
 *   - Plans (series_toolkit.py FactorPlan trees) are passed as an int32 preorder
 *     code plus a double constant pool; see INTEGRATION.md for the encoding.
 *   - Every function returns SI_OK (0) or a negative status; it never throws
 *     across the boundary.  si_last_error() returns a thread-local message.
 *   - `concurrent` != 0 maps the reference's `executor` argument
 *     (newton_schulz.py:254, richardson.py:111) to side CUDA streams joined by
 *     events; results are bitwise identical to the serial path.
 */
#ifndef SERIESINV_B200_H
#define SERIESINV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SI_OK 0
#define SI_EINVAL (-1) /* bad argument: maps to ValueError */
#define SI_ECUDA (-2)  /* CUDA launch / runtime failure: RuntimeError */
#define SI_ENOMEM (-3) /* device allocation failure: MemoryError */

#if defined(__GNUC__)
#define SI_API __attribute__((visibility("default")))
#else
#define SI_API
#endif

typedef struct si_handle_s* si_handle;
typedef struct si_comm_s* si_comm;
/* exchange callbacks of si_comm_create_callback: all-gather `count` doubles
 * per rank (rank-major into recv), in-place sum of `count` doubles; both
 * ordered on `stream` (a cudaStream_t); return 0 on success */
typedef int (*si_allgather_fn)(void* ctx, const double* send, double* recv, int64_t count,
                               void* stream);
typedef int (*si_allreduce_fn)(void* ctx, double* buf, int64_t count, void* stream);

SI_API int si_version(void);
SI_API const char* si_last_error(void);
SI_API int si_create(int device, si_handle* out);
SI_API int si_destroy(si_handle h);
/* Route the library's temporaries through a caller allocator (e.g. the host
 * framework's caching allocator) instead of the handle's stream-ordered pool.
 * alloc_fn(ctx, bytes, stream) returns device memory usable in `stream` order
 * (NULL on failure); free_fn(ctx, ptr, stream) releases it in `stream` order.
 * Pass NULL, NULL to restore the internal pool. */
SI_API int si_set_allocator(si_handle h, void* (*alloc_fn)(void* ctx, size_t bytes, void* stream),
                            void (*free_fn)(void* ctx, void* ptr, void* stream), void* ctx);
/* Release cached pool memory back to the device. */
SI_API int si_trim(si_handle h);

/* ---------------- GEMM seam (matrix_core.py:101-114) ---------------- */

/* D = alpha*(A@B) + beta*C + diag*I with A m x k, B k x n, C/D m x n.
 * One counted product (mvm if is_mv, else mmm).  Replaces mat_mul / mat_vec
 * plus the element-wise op that follows it at the reference call site
 * (e.g. `eye - mat_mul(x, a)` = alpha -1, diag 1; `mat_mul(y, z) + x` = beta 1). */
SI_API int si_gemm(si_handle h, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
            int64_t lda, const double* B, int64_t ldb, double beta, const double* C, int64_t ldc,
            double diag, double* D, int64_t ldd, int is_mv, int64_t* counters, void* stream);

/* si_gemm with the diag*I term placed at (i, i + diag_offset): used on row
 * blocks [r0, r0+m) of a block-row sharded matrix (diag_offset = r0). */
SI_API int si_gemm_ex(si_handle h, int64_t m, int64_t n, int64_t k, double alpha,
                      const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                      const double* C, int64_t ldc, double diag, int64_t diag_offset, double* D,
                      int64_t ldd, int is_mv, int64_t* counters, void* stream);

/* ---------------- sharded exchange over peer memory -----------
 * The reference has no multi-GPU layer; these replace the all-gather of a
 * row-sharded right operand (the exchange step of every `mat_mul(y, x)`
 * with x sharded, matrix_core.py:101-106) by copy-engine transfers between
 * IPC-mapped buffers plus flags, so the consuming product starts on the panels
 * that have arrived. */

/* si_gemm_ex whose k rows of B are split into npanels (<= 16) row
 * panels [panel_bounds[p], panel_bounds[p+1]) (panel_bounds[0] = 0,
 * panel_bounds[npanels] = k): rows of panel p are read only once
 * ready_flags[p] >= epoch (wrap-safe).  The DMMA kernel gates its TMA loads
 * per panel; other kernels wait on the stream.  npanels = 0: ungated.  The
 * flags must be raised by work that needs no SM (copy engines, stream memory
 * operations): the gated kernel may occupy every SM while it waits. */
SI_API int si_gemm_panels(si_handle h, int64_t m, int64_t n, int64_t k, double alpha,
                          const double* A, int64_t lda, const double* B, int64_t ldb,
                          double beta, const double* C, int64_t ldc, double diag,
                          int64_t diag_offset, double* D, int64_t ldd,
                          const uint32_t* ready_flags, uint32_t epoch,
                          const int64_t* panel_bounds, int npanels, int is_mv,
                          int64_t* counters, void* stream);

/* Exchange buffer: cudaMalloc'd (zeroed) device memory and its 64-byte CUDA IPC
 * handle, to be opened by the peer processes with si_sym_open. */
SI_API int si_sym_alloc(si_handle h, size_t bytes, void** ptr, unsigned char handle_out[64]);
SI_API int si_sym_free(si_handle h, void* ptr);
SI_API int si_sym_open(si_handle h, const unsigned char handle[64], void** ptr);
SI_API int si_sym_close(si_handle h, void* ptr);

/* Stream memory operations (no SM involved): *addr = value once the stream's
 * prior work is complete and visible; block the stream until
 * (int32_t)(*addr - value) >= 0.  addr may be a peer (IPC) mapping. */
SI_API int si_stream_write_u32(si_handle h, uint32_t* addr, uint32_t value, void* stream);
SI_API int si_stream_wait_u32(si_handle h, const uint32_t* addr, uint32_t value, void* stream);

/* Stream-ordered copy (copy engine; either side may be a peer mapping). */
SI_API int si_copy_async(si_handle h, void* dst, const void* src, size_t bytes, void* stream);

/* D = cdiag*I + sum_i coefs[i]*X[i] (nterms <= 6), one rounding per term in
 * order: the `Lin` instruction (series_toolkit.py:375-378). */
SI_API int si_lincomb(si_handle h, int64_t m, int64_t n, double cdiag, int nterms, const double* coefs,
               const double* const* X, const int64_t* ldx, double* D, int64_t ldd, void* stream);

/* si_lincomb with cdiag*I placed at (i, i + diag_offset) (row blocks). */
SI_API int si_lincomb_ex(si_handle h, int64_t m, int64_t n, double cdiag, int64_t diag_offset,
                         int nterms, const double* coefs, const double* const* X,
                         const int64_t* ldx, double* D, int64_t ldd, void* stream);

/* Host-returning reductions (synchronise `stream`): matrix_core.py:154-172. */
SI_API int si_fro_norm(si_handle h, int64_t m, int64_t n, const double* X, int64_t ldx, double* out,
                void* stream);
SI_API int si_inf_norm(si_handle h, int64_t m, int64_t n, const double* X, int64_t ldx, double* out,
                void* stream);

/* ---------------- splittings (splitting.py:101-146) ---------------- */

/* precond = I/alpha, residual = I - A/alpha  (split_scalar, splitting.py:138-140) */
SI_API int si_split_scalar(si_handle h, int64_t n, const double* A, double alpha, double* precond,
                    double* residual, void* stream);
/* precond = diag(1/d), residual = I - A/d[:,None]  (split_diagonal, splitting.py:113-114) */
SI_API int si_split_diagonal(si_handle h, int64_t n, const double* A, double* precond, double* residual,
                      void* stream);
/* out = (A + A^T)/2  (splitting.py:73) */
SI_API int si_symmetrize(si_handle h, int64_t n, const double* A, double* out, void* stream);

/* Fused symmetry check + symmetrize (splitting.py:67-73, _check_symmetric):
 * out = (A + A^T)/2 (out may equal A) in one pass over tile pairs, and the
 * host scalars asym_fro = ||A - A^T||_F, fro = ||A||_F, nonfinite = number of
 * non-finite entries (fixed-order reductions; synchronises `stream`).  The
 * caller applies the reference's test asym_fro > 1e-10 max(fro, 1e-300). */
SI_API int si_symmetrize_checked(si_handle h, int64_t n, const double* A, double* out,
                                 double* asym_fro, double* fro, double* nonfinite, void* stream);
/* is_positive_definite (splitting.py:76-98): Cholesky of (A + A^T)/2 with the
 * pivot floor d <= tol -> not PD; tol = 1e-12 ||A||_inf when default_tol != 0,
 * else pivot_tol.  Blocked (128-wide panels) with the trailing updates on the
 * DMMA GEMM; A is not modified (a workspace copy is factored).  *is_pd = 1/0;
 * on failure fail_index / fail_pivot (may be NULL) give the first failing
 * pivot.  Synchronises `stream`. */
SI_API int si_is_positive_definite(si_handle h, int64_t n, const double* A, int64_t lda,
                                   double pivot_tol, int default_tol, int* is_pd,
                                   int64_t* fail_index, double* fail_pivot, void* stream);
/* Norm-ratio power iteration (matrix_core.py:183-239, spectral_radius) from
 * the unit start vector x (device, n; overwritten with the current iterate):
 * y = A x, est = ||y||, the reference's stop rule (|est - prev| <= tol est on
 * 3 consecutive iterations), x = y / est -- all on the device; the host looks
 * at the state every `check_every` iterations (one synchronisation each).
 * *status: 1 converged (*est), 2 est == 0 (x in the null space: the caller
 * restarts with a fresh vector, as the reference does), 3 max_iter reached
 * (*best = last estimate).  *iters = iterations executed (<= max_iter). */
SI_API int si_power_iterate(si_handle h, int64_t n, const double* A, int64_t lda, double* x,
                            double tol, int64_t max_iter, int check_every, double* est,
                            double* best, int64_t* iters, int* status, void* stream);

/* Build tooling (host only, no device needed): the C++ source of the
 * compile-time program of the config-2 resident kernel for this recipe
 * (tools/gen_resident_fixed.py writes it to csrc/resident_fixed_c2.inc).
 * *len = length; written to out when cap > *len. */
SI_API int si_resident_program_source(int64_t n, int nrates, const int32_t* rates,
                                      const int32_t* plans, const int64_t* plan_offsets,
                                      const double* consts, int64_t nconsts, int order_n,
                                      char* out, int64_t cap, int64_t* len);

/* ... and of the config-1 cluster kernel (NS order `order`, 32 < n <= 64,
 * `cluster` CTAs per system; csrc/resident_fixed_c1.inc). */
SI_API int si_resident_program_source_ns(int64_t n, int order, int cluster, char* out,
                                         int64_t cap, int64_t* len);

/* ---------------- block-row sharded steps (several GPUs) ----------------
 * One rank per GPU.  Every state matrix (G, F, L, R, omega, N) is split into
 * contiguous row blocks -- rank r owns rows [r0, r1) of the near-equal split
 * returned by si_comm_rows (the first n % nranks blocks one row longer) --
 * and is passed as that block (r1 - r0 rows, contiguous).  A, S^-1, B, b and
 * theta are replicated (full n rows on every rank).  Products compute the
 * local rows; a sharded right operand is all-gathered first (one exchange per
 * state x state product: the C4 composite step has 11, as sharded.py).  The
 * GEMM DAG, the counters and every result bit equal the single-GPU entry
 * points (the per-tile K order does not depend on the split).  Every rank must
 * make the same sequence of calls (the exchanges are collective).
 * Replaces the Python block-row engine's orchestration (sharded.py), with the
 * reference's steps (newton_schulz.py:150-228, richardson.py:111-189). */
/* NCCL communicator (libnccl.so.2 is loaded on first use): rank 0 makes the id
 * with si_comm_unique_id and shares it with the other ranks (out of band). */
SI_API int si_comm_unique_id(unsigned char id[128]);
SI_API int si_comm_create_nccl(si_handle h, int nranks, int rank, const unsigned char id[128],
                               int64_t n, si_comm* out);
/* caller-provided exchange (an MPI layer, a host transport, tests) */
SI_API int si_comm_create_callback(int nranks, int rank, int64_t n, si_allgather_fn allgather,
                                   si_allreduce_fn allreduce, void* ctx, si_comm* out);
SI_API int si_comm_destroy(si_comm c);
/* this rank's rows and the exchange totals so far (any pointer may be NULL) */
SI_API int si_comm_rows(si_comm c, int64_t* r0, int64_t* r1, int64_t* gathers,
                        int64_t* bytes_received);
/* ns_step (newton_schulz.py:150-174) on row blocks */
SI_API int si_sharded_ns_step(si_handle h, si_comm comm, int64_t n, const double* a,
                              const double* g_rows, const double* f_rows, int order,
                              const int32_t* plan, int64_t plan_len, const double* consts,
                              int64_t nconsts, double* g_out_rows, double* f_out_rows,
                              int64_t* counters, void* stream);
/* composite_step (newton_schulz.py:177-228) on row blocks (serial part order) */
SI_API int si_sharded_composite_step(si_handle h, si_comm comm, int64_t n, const double* a,
                                     const double* g_rows, const double* f_rows,
                                     const double* precond, const double* residual,
                                     const double* split_matrix, int nrates, const int32_t* rates,
                                     const int32_t* plans, const int64_t* plan_offsets,
                                     const double* consts, int64_t nconsts, int order_n,
                                     double* g_out_rows, double* f_out_rows, int64_t* counters,
                                     void* stream);
/* richardson_recursive_step (richardson.py:111-189) on row blocks; theta_out
 * (n x nrhs) is replicated on return */
SI_API int si_sharded_richardson_recursive_step(
    si_handle h, si_comm comm, int64_t n, int64_t nrhs, const double* a, const double* b,
    const double* theta, const double* g_rows, const double* f_rows, const double* l_rows,
    const double* r_rows, const double* omega_rows, const double* ns_rows, int order,
    const int32_t* factor_plan, int64_t plan_len, const double* consts, int64_t nconsts,
    int doubling_sum, double* g_out_rows, double* f_out_rows, double* l_out_rows,
    double* r_out_rows, double* omega_out_rows, double* ns_out_rows, double* theta_out,
    int64_t* counters, void* stream);
/* theta - P (A theta - b) with P row-sharded; theta_out replicated on return */
SI_API int si_sharded_plain_richardson(si_handle h, si_comm comm, int64_t n, int64_t nrhs,
                                       const double* a, const double* b, const double* theta,
                                       const double* p_rows, double* theta_out, int64_t* counters,
                                       void* stream);
/* ||X||_F of a row-sharded n x cols matrix (the stop rule newton_schulz.py:328-331):
 * local sums of squares + one all-reduce; synchronises `stream` */
SI_API int si_sharded_fro_norm(si_handle h, si_comm comm, int64_t n, int64_t cols,
                               const double* x_rows, double* out, void* stream);

/* ---------------- evaluators (series_toolkit.py:279-457) ---------------- */

/* horner_eval (series_toolkit.py:279-302).  y may be NULL iff form_y; with
 * form_y the effective Y = I - X A is formed (one product) and, when y is
 * given, checked against it (SI_EINVAL on mismatch; synchronises). */
SI_API int si_horner_eval(si_handle h, int64_t n, const double* y, const double* x, int order,
                   const double* a, int form_y, double* out, int64_t* counters, void* stream);
/* factored_eval (series_toolkit.py:326-356) */
SI_API int si_factored_eval(si_handle h, int64_t n, const double* y, const double* x, const double* a,
                     int p, int w, int form_y, double* out, int64_t* counters, void* stream);
/* nested_eval (series_toolkit.py:408-429) */
SI_API int si_nested_eval(si_handle h, int64_t n, const double* y, const double* x, const double* a,
                   const int32_t* plan, int64_t plan_len, const double* consts, int64_t nconsts,
                   int form_y, double* out, int64_t* counters, void* stream);
/* geometric_apply (series_toolkit.py:432-457); base_plan = plan_order(b) for the
 * order b <= 64 reached from `order` by repeated halving (unused when b == 1). */
SI_API int si_geometric_apply(si_handle h, int64_t n, const double* y, const double* x, int order,
                       const double* a, const int32_t* base_plan, int64_t plan_len,
                       const double* consts, int64_t nconsts, double* out, int64_t* counters,
                       void* stream);
/* mat_pow_counted (matrix_core.py:137-151) */
SI_API int si_mat_pow_counted(si_handle h, int64_t n, const double* y, int e, double* out,
                       int64_t* counters, void* stream);

/* ---------------- Newton-Schulz steps (newton_schulz.py) ---------------- */

/* Fused stop-rule norm (converged, newton_schulz.py:328-331 over fro_norm,
 * matrix_core.py:167-168): the NEXT step call on this handle (si_initial_series,
 * si_ns_step*, si_composite_step*, si_composite_apply, si_initial_double,
 * si_double_ns_step) writes ||F'||_F^2 of its residual output into the device
 * double `fro2` (stream-ordered).  The products that write F' emit per-warp
 * partial sums of squares from their epilogues (FP64 GEMM, CRT of the
 * emulated products; small-n kernels one partial pass), reduced in a fixed
 * order -- deterministic, no extra pass over F'.  One-shot: the step call
 * consumes it; NULL cancels.  Not used by the si_sharded_* calls
 * (si_sharded_fro_norm). */
SI_API int si_set_step_norm(si_handle h, double* fro2);

/* initial_series (newton_schulz.py:127-147) */
SI_API int si_initial_series(si_handle h, int64_t n, const double* precond, const double* residual,
                      const double* a, int p, int w, double* g_out, double* f_out,
                      int64_t* counters, void* stream);
/* ns_step (newton_schulz.py:150-174); plan may be NULL (Horner). */
SI_API int si_ns_step(si_handle h, int64_t n, const double* a, const double* g, const double* f,
               int order, const int32_t* plan, int64_t plan_len, const double* consts,
               int64_t nconsts, double* g_out, double* f_out, int64_t* counters, void* stream);
/* si_ns_step with inputs still in flight: input_ready_events (may be NULL, or
 * 3 cudaEvent_t, each may be NULL) = {a, g, f}; the step makes its stream wait
 * on an input's event right before the first kernel that reads it, and
 * records g_done_event (may be NULL) once G' is final, before F' = I - G'A. */
SI_API int si_ns_step_ex(si_handle h, int64_t n, const double* a, const double* g,
                         const double* f, int order, const int32_t* plan, int64_t plan_len,
                         const double* consts, int64_t nconsts, void* const* input_ready_events,
                         void* g_done_event, double* g_out, double* f_out, int64_t* counters,
                         void* stream);
/* si_ns_step for inputs arriving in row panels (see si_composite_step_gated):
 * input_flags = 3 x 16 uint32 flags for {a, g, f}; f_chunks > 0: F' produced in
 * f_chunks row blocks, f_chunk_events[k] recorded after block k. */
SI_API int si_ns_step_gated(si_handle h, int64_t n, const double* a, const double* g,
                            const double* f, int order, const int32_t* plan, int64_t plan_len,
                            const double* consts, int64_t nconsts, const uint32_t* input_flags,
                            uint32_t epoch, int npanels, void* g_done_event,
                            void* const* f_chunk_events, int f_chunks, double* g_out,
                            double* f_out, int64_t* counters, void* stream);
/* composite_step (newton_schulz.py:177-228).  plans/plan_offsets[nrates+1]
 * hold, per rate, the geometric_apply base plan (empty for rate 1). */
SI_API int si_composite_step(si_handle h, int64_t n, const double* a, const double* g, const double* f,
                      const double* precond, const double* residual, const double* split_matrix,
                      int nrates, const int32_t* rates, const int32_t* plans,
                      const int64_t* plan_offsets, const double* consts, int64_t nconsts,
                      int order_n, int concurrent, double* g_out, double* f_out,
                      int64_t* counters, void* stream);
/* si_composite_step with host-copy overlap: input_ready_events (may be NULL;
 * entries may be NULL) are cudaEvent_t for {a, g, f, precond, residual,
 * split_matrix} that the step waits on just before each input's first use
 * (S^-1, B and the split matrix first, A at the first part residual, G and F
 * for the NS part), so copies still in flight overlap the first products;
 * g_done_event (may be NULL) is recorded once g_out is final, before the
 * last product F' = I - G' A, so g_out can be read back while it runs. */
SI_API int si_composite_step_ex(si_handle h, int64_t n, const double* a, const double* g,
                                const double* f, const double* precond, const double* residual,
                                const double* split_matrix, int nrates, const int32_t* rates,
                                const int32_t* plans, const int64_t* plan_offsets,
                                const double* consts, int64_t nconsts, int order_n,
                                int concurrent, void* const* input_ready_events,
                                void* g_done_event, double* g_out, double* f_out,
                                int64_t* counters, void* stream);

/* si_composite_step_ex for inputs that arrive in row panels (host->device
 * copies still in flight): input_flags (may be NULL) = 6 x 16 uint32 flags for
 * {a, g, f, precond, residual, split_matrix}; rows [n p / npanels,
 * n (p+1) / npanels) of input i are valid once input_flags[16 i + p] >= epoch.
 * The DMMA products gate their A-tile / B-slab loads on those flags, so the
 * first product starts while later panels are still copying.  The flags must
 * be raised by work that needs no SM (copy engines, stream memory operations):
 * gated products may occupy every SM while they wait.  f_chunks > 0: the last
 * two products, G' = t + r N and F' = I - G'A, are produced in f_chunks row
 * blocks, interleaved; f_chunk_events[k] is recorded once G' and F' rows of
 * block k are final, g_done_event after the last G' block (two products in
 * the counters).  The emulated products wait per row chunk for the first
 * product's A rows and for whole B / C operands. */
SI_API int si_composite_step_gated(si_handle h, int64_t n, const double* a, const double* g,
                                   const double* f, const double* precond,
                                   const double* residual, const double* split_matrix,
                                   int nrates, const int32_t* rates, const int32_t* plans,
                                   const int64_t* plan_offsets, const double* consts,
                                   int64_t nconsts, int order_n, int concurrent,
                                   const uint32_t* input_flags, uint32_t epoch, int npanels,
                                   void* g_done_event, void* const* f_chunk_events, int f_chunks,
                                   double* g_out, double* f_out, int64_t* counters,
                                   void* stream);
/* Opt-in hoisting (NOT the reference DAG, which recomputes the parts every
 * step): the state-independent half of composite_step (newton_schulz.py:
 * 204-216) -> T_comp, R_comp; and the state-dependent half (:218-220) that
 * consumes them: G' = T_comp + R_comp S_n(F) G, F' = I - G' A. */
SI_API int si_composite_parts(si_handle h, int64_t n, const double* a, const double* precond,
                              const double* residual, const double* split_matrix, int nrates,
                              const int32_t* rates, const int32_t* plans,
                              const int64_t* plan_offsets, const double* consts, int64_t nconsts,
                              double* t_out, double* r_out, int64_t* counters, void* stream);
SI_API int si_composite_apply(si_handle h, int64_t n, const double* a, const double* g,
                              const double* f, const double* t, const double* r, int order_n,
                              double* g_out, double* f_out, int64_t* counters, void* stream);
/* initial_double (newton_schulz.py:231-251) */
SI_API int si_initial_double(si_handle h, int64_t n, const double* precond, const double* residual,
                      const double* a, int p, int w, int order, double* g_out, double* f_out,
                      double* l_out, double* r_out, int64_t* counters, void* stream);
/* double_ns_step (newton_schulz.py:254-298) */
SI_API int si_double_ns_step(si_handle h, int64_t n, const double* a, const double* g, const double* f,
                      const double* l, const double* r, int order, int concurrent, double* g_out,
                      double* f_out, double* l_out, double* r_out, int64_t* counters,
                      void* stream);
/* additive_correction_step (newton_schulz.py:301-325) */
SI_API int si_additive_correction_step(si_handle h, int64_t n, const double* a, const double* z,
                                const double* g, int p, double* z_out, double* g_out,
                                int64_t* counters, void* stream);

/* ---------------- Richardson (richardson.py) ---------------- */

/* richardson_step (richardson.py:81-98): b, theta, theta_out are n x nrhs. */
SI_API int si_richardson_step(si_handle h, int64_t n, int64_t nrhs, const double* a, const double* b,
                       const double* theta, const double* g, const double* f, const double* l,
                       const double* r, int order, int q, double* g_out, double* f_out,
                       double* l_out, double* r_out, double* theta_out, int64_t* counters,
                       void* stream);
/* richardson_recursive_step (richardson.py:111-189).  omega/ns_part may be NULL
 * (first call).  Opt-in factorised variant (not in the reference): a non-NULL
 * factor_plan of order `order` evaluates N' and doubling_sum != 0 builds
 * S = prod_j (I + Gamma^(2^j)) (order must be a power of two). */
SI_API int si_richardson_recursive_step(si_handle h, int64_t n, int64_t nrhs, const double* a,
                                 const double* b, const double* theta, const double* g,
                                 const double* f, const double* l, const double* r,
                                 const double* omega, const double* ns_part, int order,
                                 const int32_t* factor_plan, int64_t plan_len,
                                 const double* consts, int64_t nconsts, int doubling_sum,
                                 int concurrent, double* g_out, double* f_out, double* l_out,
                                 double* r_out, double* omega_out, double* ns_out,
                                 double* theta_out, int64_t* counters, void* stream);
/* si_richardson_recursive_step with host-copy overlap (the numpy-facing call
 * at n = 32768 moves 69 GB in and 60 GB out per step).  input_ready_events
 * (may be NULL) = 9 cudaEvent_t, each may be NULL, for {a, b, theta, g, f, l,
 * r, omega, ns_part}: the step makes its stream wait on an input's event right
 * before the first kernel that reads it (inputs the DAG does not read -- g
 * and f in the steady state -- are waited for at the end of the call).
 * output_done_events (may be NULL) = 7 cudaEvent_t, each may be NULL, for
 * {l_out, r_out, g_out, f_out, ns_out, omega_out, theta_out}, recorded once
 * that output is final (in this order on the serial path), so it can be read
 * back while the remaining products run.  Same products, bitwise the plain
 * call. */
SI_API int si_richardson_recursive_step_ex(si_handle h, int64_t n, int64_t nrhs, const double* a,
                                    const double* b, const double* theta, const double* g,
                                    const double* f, const double* l, const double* r,
                                    const double* omega, const double* ns_part, int order,
                                    const int32_t* factor_plan, int64_t plan_len,
                                    const double* consts, int64_t nconsts, int doubling_sum,
                                    int concurrent, void* const* input_ready_events,
                                    void* const* output_done_events, double* g_out,
                                    double* f_out, double* l_out, double* r_out,
                                    double* omega_out, double* ns_out, double* theta_out,
                                    int64_t* counters, void* stream);
/* Plain update theta' = theta - P (A theta - b)  (ordering as
 * richardson.py:88-89). */
SI_API int si_plain_richardson(si_handle h, int64_t n, int64_t nrhs, const double* a, const double* b,
                        const double* theta, const double* p, double* theta_out,
                        int64_t* counters, void* stream);

/* ---------------- measurement ---------------- */

/* Start recording CUDA events around every large (TMA) GEMM launch and
 * counting kernel launches made through this handle. */
SI_API int si_profile_begin(si_handle h);
/* Stop recording; synchronises and returns the summed device time (ms) and
 * algorithmic FLOPs of the recorded TMA GEMM launches, their count, and the
 * total number of kernels this handle launched since si_profile_begin. */
SI_API int si_profile_end(si_handle h, double* gemm_ms, double* gemm_flops,
                          int64_t* gemm_launches, int64_t* total_launches);
/* FP64 DMMA (m8n8k4) register-only throughput of this device in TFLOP/s:
 * the roofline denominator (MEASURED_PEAKS.json has no FP64 entry). */
SI_API int si_dmma_peak(si_handle h, int iters, double* tflops);

/* ---------------- FP64 product backend ---------------- */

/* Which tensor-core path computes the handle's FP64 products (every n x n
 * product of the steps above; mat_mul, matrix_core.py:101-106):
 *   SI_GEMM_DMMA      FP64 DMMA (mma.sync m8n8k4), the default;
 *   SI_GEMM_OZAKI_I8  Ozaki scheme II: the product computed exactly from
 *                     power-of-two-scaled integer images of A and B, one INT8
 *                     tcgen05 GEMM per modulus (nmoduli of 256, 255, 253, ...),
 *                     recombined by the Chinese remainder theorem; used for
 *                     products whose dimensions are all >= min_dim and K <=
 *                     65536 (smaller products and GEMVs stay on DMMA; inputs
 *                     still being copied are awaited on the stream, per row
 *                     chunk for the rows of A).
 * nmoduli = 0 / min_dim = 0 keep the current value (defaults 16 / 1024).
 * The emulated result is deterministic but not bitwise the DMMA result; each
 * entry of A (B) is kept to 2^-pa (2^-pb) relative to the largest entry of its
 * row (column), pa = 55 and pb = 54 at K = 16384 with 16 moduli, and the
 * integer product is exact (ozaki.cu). */
#define SI_GEMM_DMMA 0
#define SI_GEMM_OZAKI_I8 1
SI_API int si_set_gemm_backend(si_handle h, int backend, int nmoduli, int64_t min_dim);
SI_API int si_get_gemm_backend(si_handle h, int* backend, int* nmoduli, int64_t* min_dim);
/* Workspace bound of the emulated products: D is processed in chunks of at
 * most max_rows x max_cols (rounded down to multiples of 256; 0 = automatic:
 * all rows, and <= 10 GiB of B-side and result planes per column chunk).  The
 * A-side planes are built once per row chunk, the B-side planes once per
 * product when one column chunk covers D, else per (row, column) chunk.  When
 * the allocator cannot serve a product's workspace the library retries with
 * halved chunks.  Results do not depend on the chunking (bitwise). */
SI_API int si_set_ozaki_chunks(si_handle h, int64_t max_rows, int64_t max_cols);
/* INT8 tensor-core kernel of the emulated products: 0 = automatic, 1 = CTA
 * pairs (tcgen05.mma.cta_group::2, 256 x 256 tiles), 2 = single CTAs
 * (cta_group::1, 128 x 256 tiles), 3 = single-CTA MMAs on 2-CTA clusters that
 * multicast the shared B tile.  Results are identical (exact integers). */
SI_API int si_set_ozaki_kernel(si_handle h, int variant);
/* Tuning hook of the INT8 kernels (process-wide; measurement tools):
 * rasterisation group in row tiles (0 keeps), L2 policy of the CTA-pair
 * kernel's A / B operand loads (0 evict_normal, 1 evict_last, 2 evict_first;
 * -1 keeps). */
SI_API int si_ozaki_tune(int group_m, int l2_a, int l2_b);
/* Tuning hook: shared-memory ring depth of the CTA-pair kernel (3..6). */
SI_API int si_ozaki_tune_stages(int stages);
/* Tuning hook: the longest K range one launch of the single-CTA INT8 kernel
 * covers; longer products run as several launches that accumulate the
 * residues (bitwise the unsplit result).  0 = never split (the default: the
 * split was measured at K = 32768 and lost); a multiple of 128. */
SI_API int si_ozaki_tune_ksplit(int64_t kmax);
/* The first n moduli of the emulation. */
SI_API int si_ozaki_moduli(int n, uint32_t* moduli);
/* The INT8 tensor-core kernel alone (test hook): r[l] = (a[l] @ bt[l]^T) mod
 * m_l for l < nplanes; a[l]: m x kp int8, bt[l]: n x kp int8 (row-major, kp a
 * multiple of 128), r[l]: m x n uint8; the kernel si_set_ozaki_kernel selected. */
SI_API int si_i8_gemm_mod(si_handle h, const int8_t* a, const int8_t* bt, uint8_t* r, int64_t m,
                          int64_t n, int64_t kp, int nplanes, void* stream);
/* Summed device time (ms) and int8 operations of the INT8 tensor-core kernel
 * launches recorded since si_profile_begin (emulated products only). */
SI_API int si_profile_i8(si_handle h, double* ms, double* ops, int64_t* launches);

/* ---------------- batched small systems (BASELINE config 2) ---------------- */

/* `iters` x { plain Richardson with P_k; composite_step(rates, order_n) } for
 * `batch` independent n x n systems (n <= 64), everything resident on chip.
 * A, P (in/out), F (in/out): batch x n x n; b, theta (in/out): batch x n.
 * precond/residual: batch x n x n splitting of each A; plans as in
 * si_composite_step.  Counters are per system (identical for all systems). */
SI_API int si_batched_composite_richardson(si_handle h, int64_t batch, int64_t n, const double* a,
                                    const double* b, const double* precond,
                                    const double* residual, int nrates, const int32_t* rates,
                                    const int32_t* plans, const int64_t* plan_offsets,
                                    const double* consts, int64_t nconsts, int order_n,
                                    int iters, double* p_io, double* f_io, double* theta_io,
                                    int64_t* counters, void* stream);
/* The same with separate inputs and outputs (the caller keeps its inputs:
 * the reference's steps are pure, newton_schulz.py:58-72); in == out is
 * allowed and equals si_batched_composite_richardson. */
SI_API int si_batched_composite_richardson_ex(
    si_handle h, int64_t batch, int64_t n, const double* a, const double* b, const double* precond,
    const double* residual, int nrates, const int32_t* rates, const int32_t* plans,
    const int64_t* plan_offsets, const double* consts, int64_t nconsts, int order_n, int iters,
    const double* p_in, const double* f_in, const double* theta_in, double* p_out, double* f_out,
    double* theta_out, int64_t* counters, void* stream);
/* si_batched_composite_richardson_ex for inputs that arrive by chunks of
 * `chunk` systems (host->device copies in flight): system i's inputs are read
 * once chunk_ready[i / chunk] >= epoch (wrap-safe); chunk_done (may be NULL)
 * gets +1 per finished system of each chunk, after its outputs are written, so
 * a copy stream can wait (si_stream_wait_u32) and read a chunk back early.
 * Flags must be raised by work that needs no SM (copy engines, stream memory
 * operations). */
SI_API int si_batched_composite_richardson_gated(
    si_handle h, int64_t batch, int64_t n, const double* a, const double* b, const double* precond,
    const double* residual, int nrates, const int32_t* rates, const int32_t* plans,
    const int64_t* plan_offsets, const double* consts, int64_t nconsts, int order_n, int iters,
    const double* p_in, const double* f_in, const double* theta_in, double* p_out, double* f_out,
    double* theta_out, const uint32_t* chunk_ready, uint32_t epoch, int64_t chunk,
    uint32_t* chunk_done, int64_t* counters, void* stream);

/* BASELINE config 1 shape (batch = 1, n <= 64) and batches of it: `iters` x
 * { plain Richardson with P_k; ns_step(order, plan) } with the state resident
 * in shared memory (one launch for the whole run).  A: batch x n x n; P, F
 * (in/out): batch x n x n; b, theta (in/out): batch x n; plan may be NULL. */
SI_API int si_batched_ns_richardson(si_handle h, int64_t batch, int64_t n, const double* a,
                                    const double* b, int order, const int32_t* plan,
                                    int64_t plan_len, const double* consts, int64_t nconsts,
                                    int iters, double* p_io, double* f_io, double* theta_io,
                                    int64_t* counters, void* stream);
/* Separate inputs and outputs (in == out allowed). */
SI_API int si_batched_ns_richardson_ex(si_handle h, int64_t batch, int64_t n, const double* a,
                                       const double* b, int order, const int32_t* plan,
                                       int64_t plan_len, const double* consts, int64_t nconsts,
                                       int iters, const double* p_in, const double* f_in,
                                       const double* theta_in, double* p_out, double* f_out,
                                       double* theta_out, int64_t* counters, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SERIESINV_B200_H */
