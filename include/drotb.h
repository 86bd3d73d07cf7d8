/* drotb.h -- C ABI of libdrotb200.so, the B200-native DROT solver.
 *
 * This is the drop-in boundary for the reference's solve path.  The
 * reference (/root/reference/proj/core) is a header-only C++20 template
 * library with no C ABI; each entry point below replaces one reference
 * interface, cited as file:line under proj/core/include/drot/:
 *
 *   drotb_solve_f32/_f64        drot::solve<T>            solver.hpp:372-540
 *   drotb_step_f32/_f64         drot::drot_step<T>        solver.hpp:361-370
 *   drotb_engine_*              drot::FusedEngine<T>      fused.hpp:107-202
 *     drotb_engine_pass_f32/_f64   fused_pass :127-134 / fused_pass_skip_cost
 *                                  :140-155 / unfused_pass :359-531
 *   drotb_check_problem_f32/_f64 drot::check_problem      problem.hpp:122-136
 *   drotb_check_problem_tol_*   check_problem(pr, simplex_tol) problem.hpp:122-124
 *   drotb_materialize_plan_*    drot::materialize_plan<T> solver.hpp:204-217
 *   drotb_materialize_y_*       drot::materialize_y<T>    solver.hpp:221-230
 *   drotb_gen_gaussian          drot::gen_gaussian_problem probgen.hpp:131-170
 *   drotb_config_default        drot::DrotConfig{}        solver.hpp:51-88
 *   drotb_errc_name             drot::errc_name           errors.hpp:48-73
 *
 * Conventions (all functions):
 *   - plain pointers and sizes only; matrices are column-major m x n
 *     (element (i,j) at [j*m + i], matrix.hpp:56-59), contiguous;
 *   - host pointers unless the name says _dev;
 *   - return 0 on success, otherwise 1 + the ordinal of drot::Errc
 *     (errors.hpp:24-46), or a value >= DROTB_ERR_CUDA for CUDA/NCCL failures;
 *     drotb_last_error() returns "<errc_name>: <what>" exactly like
 *     drot::fail (errors.hpp:86-88).  Nothing throws across the ABI;
 *   - divergence is a status (DROTB_NUMERICAL_FAILURE) in drotb_solve_*, and
 *     an error (non_finite_iterate) in drotb_step_*, as in the reference.
 */
#ifndef DROTB_H_
#define DROTB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DROTB_ABI_VERSION 1

/* drot::Errc ordinals (errors.hpp:24-46); return codes are 1 + these. */
enum drotb_errc {
  DROTB_ERRC_NEGATIVE_COST = 0,
  DROTB_ERRC_MARGINAL_NOT_SIMPLEX = 1,
  DROTB_ERRC_EMPTY_DIMENSION = 2,
  DROTB_ERRC_NON_FINITE_ENTRY = 3,
  DROTB_ERRC_SHAPE_MISMATCH = 4,
  DROTB_ERRC_NON_POSITIVE_RHO = 5,
  DROTB_ERRC_INVALID_INITIAL_PLAN = 6,
  DROTB_ERRC_NON_FINITE_ITERATE = 7,
  DROTB_ERRC_ZERO_MARGINAL = 8,
  DROTB_ERRC_TOO_LARGE = 9,
  DROTB_ERRC_DEGENERATE_COST = 10,
  DROTB_ERRC_DIMENSION_MISMATCH = 11,
  DROTB_ERRC_FOLD_STATE_MISMATCH = 12,
  DROTB_ERRC_BAD_CONFIG = 20
};
#define DROTB_ERR_CUDA 1000 /* CUDA runtime / driver failure */
#define DROTB_ERR_NCCL 2000 /* NCCL failure */

/* drot::SolveStatus (problem.hpp:66). */
enum drotb_status {
  DROTB_CONVERGED = 0,
  DROTB_MAX_ITERS = 1,
  DROTB_NUMERICAL_FAILURE = 2
};

/* drot::EngineKind (solver.hpp:37-40). */
enum drotb_engine_kind { DROTB_ENGINE_REFERENCE = 0, DROTB_ENGINE_FUSED = 1 };

/* Reduction order of the device kernels (B200 extension; no reference
 * counterpart).
 *   DROTB_ORDER_REFERENCE: reproduce the reference's deterministic reduction
 *     tree exactly (plan_tiles(bs=64, ws) order, tiles.cpp:20-47, merged as
 *     fused.hpp:312-329; sequential vec_sum/vec_norm_sq, matrix.hpp:99-118;
 *     sequential double chains in solver.hpp:312-354, 443-490).  Iterates,
 *     duals, gate decisions and iteration counts are bitwise those of
 *     drot::solve<T> with deterministic=true.  Single GPU only; slower.
 *   DROTB_ORDER_FAST: u and v stay in reference order (free in the fused
 *     sweep); scalar reductions and the O(m+n) sums use a fixed parallel
 *     tree.  Deterministic run to run and independent of the GPU count.
 */
enum drotb_order { DROTB_ORDER_REFERENCE = 0, DROTB_ORDER_FAST = 1 };

/* Mirrors drot::DrotConfig (solver.hpp:51-88) field for field, plus B200
 * extensions at the end. */
typedef struct drotb_config {
  double rho0;                 /* rho = rho0 / (m + n) */
  int32_t has_rho_override;    /* std::optional<double> rho_override */
  int32_t relative_tolerances;
  double rho_override;
  double tol_primal, tol_dual, tol_gap;
  int64_t max_iters;
  int64_t check_every;
  int32_t engine;              /* enum drotb_engine_kind */
  int32_t skip_cost;
  int32_t deterministic;
  int32_t record_trace;
  int64_t workers;             /* CPU knob: accepted, ignored */
  int64_t block_rows;          /* reduction-tree tile rows (64 reproduces bitwise) */
  int64_t work_size;           /* tile columns = work_size * block_rows */
  int64_t trace_every;
  int32_t precision;           /* 0 = f32, 1 = f64 (front-end dispatch only) */
  /* ---- B200 extensions ---- */
  int32_t device;              /* CUDA device ordinal, -1 = current */
  int32_t order;               /* enum drotb_order */
  int32_t use_graphs;          /* capture iteration pairs in CUDA graphs */
} drotb_config;

/* drot::ResidualReport (problem.hpp:57-62). */
typedef struct drotb_report {
  double r_primal, r_dual, gap, objective;
} drotb_report;

/* drot::TraceRow (problem.hpp:77-85). */
typedef struct drotb_trace_row {
  int64_t iter;
  double r_primal, r_dual, gap, objective, ergodic_objective,
      fixed_point_residual;
} drotb_trace_row;

/* Scalars of drot::FusedPassOutput<T> (fused.hpp:42-60); T widened to
 * double (exact for float). */
typedef struct drotb_pass_out {
  double cost_dot, max_abs, dual_sq, dx_sq, prev_cost_dot;
  int32_t cost_valid, nonfinite, dual_valid, dx_valid, prev_cost_valid;
  int32_t pad_;
} drotb_pass_out;

/* drot::MemoryCounters (fused.hpp:34-39). */
typedef struct drotb_counters {
  uint64_t passes, xy_elems_read, xy_elems_written, cost_elems_read;
} drotb_counters;

/* Pass kinds for drotb_engine_pass_*. */
enum drotb_pass_kind {
  DROTB_PASS_FUSED = 0,     /* fused_pass (fused.hpp:127) */
  DROTB_PASS_SKIP_COST = 1, /* fused_pass_skip_cost (fused.hpp:140) */
  DROTB_PASS_UNFUSED = 2    /* unfused_pass (fused.hpp:359) */
};

/* ---- library ------------------------------------------------------------ */
int32_t drotb_abi_version(void);
const char* drotb_last_error(void);
const char* drotb_errc_name(int32_t errc);
void drotb_config_default(drotb_config* cfg);
/* Number of device kernels launched by this process so far (diagnostic). */
int64_t drotb_kernel_launches(void);

/* ---- one-shot solve: drot::solve<T> (solver.hpp:372-540) ---------------- *
 * C (m*n), p (m), q (n), x0 (m*n or NULL): host inputs.
 * plan_out (m*n), mu_out (m), nu_out (n): host outputs (each may be NULL).
 * trace_out: up to trace_cap rows (may be NULL); *trace_len receives the
 * number of rows the solve recorded.  rho_out receives the T-precision rho
 * of the DualCertificate. */
int drotb_solve_f32(const float* C, int64_t m, int64_t n, const float* p,
                    const float* q, const drotb_config* cfg, const float* x0,
                    float* plan_out, float* mu_out, float* nu_out,
                    float* rho_out, drotb_report* report,
                    drotb_trace_row* trace_out, int64_t trace_cap,
                    int64_t* trace_len, int64_t* iterations, int32_t* status,
                    double* wall_time_s);
int drotb_solve_f64(const double* C, int64_t m, int64_t n, const double* p,
                    const double* q, const drotb_config* cfg, const double* x0,
                    double* plan_out, double* mu_out, double* nu_out,
                    double* rho_out, drotb_report* report,
                    drotb_trace_row* trace_out, int64_t trace_cap,
                    int64_t* trace_len, int64_t* iterations, int32_t* status,
                    double* wall_time_s);

/* drotb_solve_* keeps one device context per host thread and precision
 * (buffers, stream, schedule, graphs) for repeated solves of the same shape
 * and configuration; this frees it. */
void drotb_release_cache(void);

/* ---- one iteration on caller-owned state: drot::drot_step<T> ------------ *
 * (solver.hpp:361-370).  The DrotState<T> fields (solver.hpp:98-114) are
 * passed as arrays and updated in place: xy (m*n), *cost_folded, row_shift
 * (phi, m), col_shift (varphi, n), y_row_defect (a, m), y_col_defect (b, n),
 * *y_mass_gap (alpha), row_residual (r, m), col_residual (s, n),
 * *x_mass_gap (beta), *iter.  Throws (returns) non_finite_iterate on
 * overflow like the reference. */
int drotb_step_f32(float* xy, int32_t* cost_folded, float* row_shift,
                   float* col_shift, float* y_row_defect, float* y_col_defect,
                   float* y_mass_gap, float* row_residual, float* col_residual,
                   float* x_mass_gap, int64_t* iter, const float* C, int64_t m,
                   int64_t n, const float* p, const float* q,
                   const drotb_config* cfg);
int drotb_step_f64(double* xy, int32_t* cost_folded, double* row_shift,
                   double* col_shift, double* y_row_defect,
                   double* y_col_defect, double* y_mass_gap,
                   double* row_residual, double* col_residual,
                   double* x_mass_gap, int64_t* iter, const double* C,
                   int64_t m, int64_t n, const double* p, const double* q,
                   const drotb_config* cfg);
/* drot::init_state<T> (solver.hpp:143-186) into caller-owned arrays. */
int drotb_init_state_f32(float* xy, int32_t* cost_folded, float* row_shift,
                         float* col_shift, float* y_row_defect,
                         float* y_col_defect, float* y_mass_gap,
                         float* row_residual, float* col_residual,
                         float* x_mass_gap, int64_t* iter, const float* C,
                         int64_t m, int64_t n, const float* p, const float* q,
                         const float* x0, const drotb_config* cfg);
int drotb_init_state_f64(double* xy, int32_t* cost_folded, double* row_shift,
                         double* col_shift, double* y_row_defect,
                         double* y_col_defect, double* y_mass_gap,
                         double* row_residual, double* col_residual,
                         double* x_mass_gap, int64_t* iter, const double* C,
                         int64_t m, int64_t n, const double* p,
                         const double* q, const double* x0,
                         const drotb_config* cfg);
/* ---- engine: drot::FusedEngine<T> (fused.hpp:107-202) ------------------- */
typedef struct drotb_engine drotb_engine;
/* plan_tiles(m, n, block_rows, work_size, workers) (tiles.cpp:20-47);
 * precision 0 = f32, 1 = f64; device -1 = current. */
int drotb_engine_create(drotb_engine** eng, int64_t m, int64_t n,
                        int64_t block_rows, int64_t work_size,
                        int32_t precision, int32_t device);
void drotb_engine_destroy(drotb_engine* eng);
/* One pass on host arrays.  kind: enum drotb_pass_kind.  For
 * DROTB_PASS_SKIP_COST, *cost_folded is the FusedArray fold state (in/out)
 * and fold the requested direction (mismatch -> fold_state_mismatch,
 * fused.hpp:146-149); otherwise both are ignored.  row_sums (m) / col_sums
 * (n) receive u = X+ e and v = X+' f.  counters (may be NULL) are
 * incremented exactly as the reference's MemoryCounters. */
int drotb_engine_pass_f32(drotb_engine* eng, float* xy, const float* C,
                          const float* row_shift, const float* col_shift,
                          float rho, int32_t kind, int32_t fold,
                          int32_t* cost_folded, int32_t parity,
                          int32_t want_dual, int32_t want_dx,
                          int32_t deterministic, float* row_sums,
                          float* col_sums, drotb_pass_out* out,
                          drotb_counters* counters);
int drotb_engine_pass_f64(drotb_engine* eng, double* xy, const double* C,
                          const double* row_shift, const double* col_shift,
                          double rho, int32_t kind, int32_t fold,
                          int32_t* cost_folded, int32_t parity,
                          int32_t want_dual, int32_t want_dx,
                          int32_t deterministic, double* row_sums,
                          double* col_sums, drotb_pass_out* out,
                          drotb_counters* counters);

/* ---- validation / diagnostics ------------------------------------------- */
int drotb_check_problem_f32(const float* C, int64_t m, int64_t n,
                            const float* p, const float* q);
int drotb_check_problem_f64(const double* C, int64_t m, int64_t n,
                            const double* p, const double* q);
/* check_problem(problem, simplex_tol) (problem.hpp:122-124): the same scan
 * with the caller's |sum - 1| tolerance (the two functions above use the
 * reference default 1e-12).  validate_problem's renormalize option
 * (problem.hpp:141-154) is O(m+n) host work in the front ends, followed by
 * this check. */
int drotb_check_problem_tol_f32(const float* C, int64_t m, int64_t n,
                                const float* p, const float* q, double simplex_tol);
int drotb_check_problem_tol_f64(const double* C, int64_t m, int64_t n,
                                const double* p, const double* q, double simplex_tol);

/* materialize_plan (solver.hpp:204-217) / materialize_y (:221-230) of a
 * caller-owned DrotState array xy (m*n; holds X - rho C when cost_folded):
 * plan = max(xy + rho*C, 0) when folded, else xy; y = plan + (phi_i +
 * varphi_j).  C may be NULL when cost_folded == 0.  Evaluated on the device. */
int drotb_materialize_plan_f32(const float* xy, int32_t cost_folded, const float* C,
                               int64_t m, int64_t n, float rho, float* plan);
int drotb_materialize_plan_f64(const double* xy, int32_t cost_folded, const double* C,
                               int64_t m, int64_t n, double rho, double* plan);
int drotb_materialize_y_f32(const float* xy, int32_t cost_folded, const float* C,
                            const float* row_shift, const float* col_shift, int64_t m,
                            int64_t n, float rho, float* y);
int drotb_materialize_y_f64(const double* xy, int32_t cost_folded, const double* C,
                            const double* row_shift, const double* col_shift, int64_t m,
                            int64_t n, double rho, double* y);

/* residual_report (problem.hpp:174-225) of an arbitrary (plan, cert) pair,
 * evaluated on the device: plan (m*n), mu (m), nu (n) host arrays.
 * exact != 0 evaluates every sum in the reference's order (bitwise equal
 * report, serial chains); exact == 0 uses fixed parallel trees. */
int drotb_residual_report_f32(const float* C, int64_t m, int64_t n, const float* p,
                              const float* q, const float* plan, const float* mu,
                              const float* nu, int32_t exact, drotb_report* out);
int drotb_residual_report_f64(const double* C, int64_t m, int64_t n, const double* p,
                              const double* q, const double* plan, const double* mu,
                              const double* nu, int32_t exact, drotb_report* out);

/* ---- Sinkhorn baseline: drot::sinkhorn_solve<T> (reference.hpp:165-288) --
 * The paper's comparison method on the B200 (plain Sinkhorn on
 * K = exp(-C/eta)); errors: bad_config (eta <= 0), zero_marginal (p or q has
 * a non-positive entry).  Divergence is a status (numerical_failure, zero
 * plan/duals, NaN report).  trace rows: one per check (r_primal = the
 * marginal error, r_dual = -1 = kResidualNotApplicable).  exact_report
 * selects the reference-order residual_report. */
int drotb_sinkhorn_f32(const float* C, int64_t m, int64_t n, const float* p, const float* q,
                       float eta, double tol, int64_t max_iters, int64_t check_every,
                       int32_t exact_report, float* plan, float* mu, float* nu,
                       drotb_report* report, drotb_trace_row* trace, int64_t trace_cap,
                       int64_t* trace_len, int64_t* iterations, int32_t* status, double* wall);
int drotb_sinkhorn_f64(const double* C, int64_t m, int64_t n, const double* p, const double* q,
                       double eta, double tol, int64_t max_iters, int64_t check_every,
                       int32_t exact_report, double* plan, double* mu, double* nu,
                       drotb_report* report, drotb_trace_row* trace, int64_t trace_cap,
                       int64_t* trace_len, int64_t* iterations, int32_t* status, double* wall);
/* Device time (ms, CUDA events) of the iteration loop of this host thread's
 * last drotb_sinkhorn_* call -- the batches of sweeps, updates and checks,
 * without the uploads, the kernel build and the final plan (B200 extension). */
double drotb_sinkhorn_last_loop_ms(void);

/* ---- problem generation (probgen.hpp:131-170, host, bit-identical) ------ *
 * Writes C (m*n column-major, normalized to max 1), p (m), q (n) in double.
 * dirichlet != 0 selects Dirichlet(1..1) marginals (probgen.hpp:115-127). */
int drotb_gen_gaussian(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                       int32_t dirichlet, double* C, double* p, double* q);
/* Same instance cast to float (gen_gaussian_problem_as<float>,
 * probgen.hpp:172-180); multi-threaded, never materializes the double
 * matrix. */
int drotb_gen_gaussian_f32(int64_t m, int64_t n, double sigma_t,
                           uint64_t seed, float* C);
/* lo + (hi - lo) * CounterRng(seed).next_unit() for outputs 1..count
 * (rng.hpp:49-57): the reference's random_matrix fixture in storage order
 * (tests/support/oracles.hpp:128-135), used for the C1 / C3 cost matrices. */
int drotb_counter_uniform(uint64_t seed, int64_t count, double lo, double hi,
                          double* out);
/* Simplex vector of exact dyadic entries k_i * 2^-K summing to exactly 1,
 * as uniform as the format allows (the inputs the reference's 1e-12 simplex
 * check accepts at every size; B200 extension). */
int drotb_dyadic_marginal_f32(int64_t len, float* out);
int drotb_dyadic_marginal_f64(int64_t len, double* out);

/* ---- session: device-resident solve for benchmarks and multi-GPU -------- *
 * A session owns device copies of C, p, q and the DrotState, a CUDA stream
 * and captured CUDA graphs.  It runs the same iteration as drotb_solve_*. */
typedef struct drotb_session drotb_session;
int drotb_session_create(drotb_session** s, int64_t m, int64_t n,
                         int32_t precision, const drotb_config* cfg);
void drotb_session_destroy(drotb_session* s);
/* Use an external CUDA stream (cudaStream_t passed as void*; NULL = own). */
int drotb_session_set_stream(drotb_session* s, void* stream);
/* Upload the problem from host (is_device == 0) or device pointers of the
 * session's precision.  Validates exactly like check_problem. */
int drotb_session_set_problem(drotb_session* s, const void* C, const void* p,
                              const void* q, int32_t is_device);
/* Generate gen_gaussian_problem(m_global, n, sigma_t, seed)'s cost ON THE
 * DEVICE (K7, bit-identical to probgen.hpp:131-180 cast to the session's
 * precision; a shard generates its rows, normalized by the global max), with
 * marginals: 0 uniform 1/m, 1 dyadic-uniform, 2 Dirichlet (probgen.hpp:
 * 115-127), 3 random_simplex(seed^0x1111 / seed^0x2222) (oracles.hpp:137-147).
 * Validates like check_problem. */
int drotb_session_gen_gaussian(drotb_session* s, double sigma_t, uint64_t seed,
                               int32_t marginals);
/* random_matrix(m_global, n, seed, lo, hi) (oracles.hpp:128-135) generated on
 * the device in the global column-major storage order; marginals as above. */
int drotb_session_gen_uniform(drotb_session* s, uint64_t seed, double lo, double hi,
                              int32_t marginals);
/* Support of the current plan (materialize_plan values, solver.hpp:204-217):
 * xmax = max x_ij and nnz = #{x_ij > max(abs_tau, rel_tau * xmax)}, over all
 * ranks when row-sharded (collective).  SURVEY §8(c) support parity. */
int drotb_session_support(drotb_session* s, double rel_tau, double abs_tau, int64_t* nnz,
                          double* xmax);
/* Profiling aid (DROTB_TAIL_STAMPS=1 at session creation): copies and resets
 * the device timeline of the solve loop, 64 iterations deep: out[3072] =
 * [slot = iteration & 63][point 0..23][min, max over CTAs] %globaltimer ns
 * (points: csrc/drotb_internal.hpp kStampPts). */
int drotb_session_tail_stamps(drotb_session* s, uint64_t* out3072);
/* Debug aid: device addresses of the book, the tail barrier words and the
 * exchange buffer, and the tail grid size. */
int drotb_session_debug_ptrs(drotb_session* s, uint64_t* out4);
/* Copy the session's (local) cost matrix to host, m x n column-major. */
int drotb_session_get_cost(drotb_session* s, void* out);
/* init_state (x0 host pointer or NULL); resets the solve bookkeeping. */
int drotb_session_init(drotb_session* s, const void* x0);
/* Enqueue up to n_iters iterations of the solve loop (gating included) on
 * the session stream; returns without synchronizing. */
int drotb_session_enqueue(drotb_session* s, int64_t n_iters);
/* Capture and instantiate (without launching) every CUDA graph that
 * drotb_session_enqueue(s, n_iters) would launch from the current state, so
 * that a timed enqueue of the same length captures nothing. */
int drotb_session_prepare(drotb_session* s, int64_t n_iters);
/* Number of CUDA graphs this session has captured and instantiated. */
int64_t drotb_session_graph_builds(drotb_session* s);
/* Run the loop to termination (converged / max_iters / failure). */
int drotb_session_run(drotb_session* s);
int drotb_session_synchronize(drotb_session* s);
/* Results of the solve so far (synchronizes). */
int drotb_session_status(drotb_session* s, int32_t* status, int64_t* iterations,
                         drotb_report* report);
int drotb_session_get_plan(drotb_session* s, void* plan_out, void* mu_out,
                           void* nu_out);
/* Device pointer of the iterate array (for tests / zero-copy consumers). */
void* drotb_session_device_xy(drotb_session* s);
void* drotb_session_stream(drotb_session* s);
/* Kernels launched per iteration and bytes moved per iteration by the pass
 * (algorithmic) for the roofline bookkeeping. */
int drotb_session_pass_bytes(drotb_session* s, double* bytes_fold,
                             double* bytes_skip);

/* Run exactly n_iters iterations eagerly, bracketed by CUDA events on the
 * session stream, with an event pair around every fused-sweep launch.
 * total_ms: first-to-last event; pass_ms: summed sweep durations; n_pass:
 * sweeps timed; pass_bytes: their algorithmic bytes (3*s*m*n per C-reading
 * sweep, 2*s*m*n per skip sweep); launches: kernels launched.
 * Synchronizes. */
int drotb_session_run_timed(drotb_session* s, int64_t n_iters, double* total_ms,
                            double* pass_ms, int64_t* n_pass, double* pass_bytes,
                            int64_t* launches);

/* ---- multi-GPU (row sharding, NCCL) ------------------------------------- */
#define DROTB_NCCL_ID_BYTES 128
/* ncclGetUniqueId for rank 0 to broadcast (e.g. over torch.distributed). */
int drotb_nccl_unique_id(char* out128);
/* Row range of `rank` in a world_size-way split of m rows: contiguous, as
 * even as possible, aligned to the sweep's 512-row CTA blocks (64 rows when
 * m < 512 * world_size).  With 512-aligned shards the peer-memory exchange
 * reproduces the one-GPU solve bit for bit. */
int drotb_shard_rows(int64_t m, int32_t world_size, int32_t rank,
                     int64_t* row_begin, int64_t* row_end);
/* A session holding rows [row_begin, row_end) of an m_global x n problem,
 * one process per GPU.  X, C, phi, a, r, p are local; varphi, b, s, q are
 * replicated.  Per iteration: one NCCL allreduce of [v partial (n) | pass
 * scalars], one of the row-side dual/trace sums, and -- only when the gate
 * fires -- one of the exact-report sums.  set_problem then
 * takes the local rows of C (row_end-row_begin x n, column-major), the local
 * p and the full q; get_plan returns the local rows.  order must be fast. */
int drotb_session_create_sharded(drotb_session** s, int64_t m_global, int64_t n,
                                 int32_t precision, const drotb_config* cfg,
                                 int32_t rank, int32_t world_size,
                                 const char* nccl_id128, int64_t row_begin,
                                 int64_t row_end);

/* The same row shard with the per-iteration exchange fused into the
 * cooperative tail kernel over NVLink peer memory (no NCCL): each rank
 * writes its column partials and scalars straight into every peer's
 * exchange buffer, raises a generation flag there, and reduces the world
 * payloads in rank order (bit-identical on every rank).  Setup collectives
 * (validation, init, confirm report) use the same buffers.  After creation,
 * exchange the buffers -- drotb_session_exchange_buffer gives this rank's
 * device pointer (peers in the same process) and CUDA IPC handle (64 bytes,
 * one process per GPU) -- then call drotb_session_attach_peers on every rank
 * with all ranks' pointers or handles (rank order; this rank's entry is
 * ignored) before set_problem / gen_*.  Every later call is collective. */
int drotb_session_create_sharded_p2p(drotb_session** s, int64_t m_global, int64_t n,
                                     int32_t precision, const drotb_config* cfg, int32_t rank,
                                     int32_t world_size, int64_t row_begin, int64_t row_end);
int drotb_session_exchange_buffer(drotb_session* s, uint64_t* dev_ptr, char* ipc_handle64);
int drotb_session_attach_peers(drotb_session* s, const uint64_t* dev_ptrs,
                               const char* ipc_handles);

#ifdef __cplusplus
}
#endif

#endif /* DROTB_H_ */
