// drotb_internal.hpp -- shared declarations of the B200 DROT engine
// (device argument blocks, solver bookkeeping, kernel launchers).
//
// Device layout (column-major like the reference, matrix.hpp:56-59):
//   X, C        ld x n, ld = round_up(m_rows, 32) (every column 128-B aligned;
//               pad rows are zero and never enter a reduction)
//   phi, a, r   ld-length row vectors;  varphi, b, s   n-length column vectors
//   ustrip      grid_cols x ld     per-tile row-sum strips  (fused.hpp:194)
//   vstrip      grid_rows64 x n    per-64-row-block column-sum strips (:195)
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace drotb {

// Pass modes of the fused sweep (fused.hpp:244-289).
enum PassMode : int {
  kPlain0 = 0,  // fused_pass, parity 0: ((x+phi)+varphi) - rho c
  kPlain1 = 1,  // fused_pass, parity 1: ((x - rho c)+phi)+varphi
  kFold = 2,    // skip-C fold pass: parity 0, writes X+ - rho C
  kSkip = 3,    // skip-C pass on a folded array: (x+phi)+varphi, no C read
};

constexpr int kWarpsPerCta = 4;
constexpr int kChunkCols = 16;   // columns staged per warp for the v sums
constexpr int kVBlockRows = 64;  // reference block_rows of the v strips

// Profiling aid (DROTB_TAIL_STAMPS=1): a %globaltimer timeline of the solve
// loop, kStampSlots iterations deep (slot = iteration & (kStampSlots - 1)),
// kStampPts points per iteration, each as a (min, max) pair over CTAs:
//   0 K1 entry, 1 K1 exit, 2 tail entry, 3 tail merge done, 4 tail release
//   (scalar section done), 5 tail update done, 6 tail exit, 7 merge strips
//   loaded, 8 merge r/s stored, 9 K1 partial slice loaded, 10 last CTA
//   knows it is last, 11 last CTA partial loads + sums done, 12 last CTA
//   scalar logic done, 13 release observed (waiting CTAs)
// fixed-point row / column sums (PassArgs::fx): value = integer * 2^-46,
// |sum| < 2^17; resolution 1.4e-14 per partial (fp32 sums of O(1e-5..1)
// entries need ~1e-12 absolute)
constexpr double kFxScale = 0x1p46;
constexpr double kFxInv = 0x1p-46;
constexpr double kFxLoScale = 0x1p86;  // fp64 remainder word
constexpr double kFxLoInv = 0x1p-86;

// Exact accumulators (one-GPU cooperative tail): every scalar sum of an
// iteration is accumulated as a pair of 64-bit integers -- hi =
// round(x * 2^42), lo = round((x - hi * 2^-42) * 2^82) -- with integer
// atomics, so the totals are exact sums of the rounded terms: independent of
// the order, the grid and the number of GPUs.  Valid for |sum| < 2^20 (every
// per-iteration sum of a solve from X0 = p q': mass, costs and residuals are
// O(1)); resolution 2^-82.
constexpr double kHiScale = 0x1p42;
constexpr double kHiInv = 0x1p-42;
constexpr double kLoScale = 0x1p82;
constexpr double kLoInv = 0x1p-82;
// accumulator words per parity: [0, 22) A: 11 sums of the sweep + merge
// {cost, prev, dual, dx, sum r, |r|^2, |s|^2, sum p a, sum p r, sum q b,
// sum q s}, [22] max |t| bits, [23] non-finite count; [24, 40) P: the 8
// update sums; [40, 44) R: the 2 confirm-report sums
enum XAcc : int {
  kXaCost = 0, kXaPrev = 1, kXaDual = 2, kXaDx = 3, kXaSumR = 4, kXaR2 = 5, kXaS2 = 6,
  kXaPA = 7, kXaPR = 8, kXaQB = 9, kXaQS = 10, kXaMax = 22, kXaBad = 23, kXaP = 24, kXaR = 40,
  kXaWords = 64
};

constexpr int kStampSlots = 64;
constexpr int kStampPts = 24;
constexpr int kStampWords = kStampSlots * kStampPts * 2;

template <class T>
struct PassPartial {  // per-CTA partial reductions (fused.hpp:85-93)
  T cost, prev, dual, dx, max_abs;
  int bad;
  int pad;
};

template <class T>
struct PassArgs {
  T* __restrict__ xy;
  const T* __restrict__ cost;
  const T* __restrict__ phi;
  const T* __restrict__ varphi;
  T rho;
  int64_t m, n, ld;     // rows, cols, leading dimension
  int64_t row_begin;    // global row of local row 0 (multi-GPU shards)
  int64_t tc;           // tile columns (ws * bs)
  T* __restrict__ ustrip;
  T* __restrict__ vstrip;
  PassPartial<T>* __restrict__ partials;
  const int* stop;      // device stop flag (nullptr: never)
  unsigned long long* stamps;  // profiling aid (DROTB_TAIL_STAMPS): device timeline, or null
  const int64_t* iter;         // Book::iter (timeline slot of this sweep)
  // fx = 1 (fp32 fast order, one GPU): the row / column sums are accumulated
  // as 64-bit fixed point (kFxScale) with integer atomics -- exact, hence
  // order-independent and deterministic -- instead of strips
  long long* ufx;
  long long* vfx;
  int32_t fx;
  int32_t pad_fx;
  long long* xacc;      // exact accumulators of this iteration (kXaWords), or null: partials
  int32_t pdl;          // launch as a programmatic dependent (after the coop tail)
  int32_t trigger;      // a programmatic dependent (the coop tail) follows: trigger early
  int32_t l2hint;       // 1: stream X / C with an L2 evict_first policy (sweep.cuh)
  int32_t pad_l2;
};

// Device-resident solver bookkeeping: every scalar of the solve loop
// (solver.hpp:394-521) and of DrotState (solver.hpp:98-114).
template <class T>
struct Book {
  // DrotState scalars
  T alpha, beta, coef;
  T nr2, ns2;  // vec_norm_sq(r), vec_norm_sq(s)
  int64_t iter;        // iterations completed (state.iter)
  int64_t iterations;  // result.trace.iterations
  int32_t folded;
  int32_t stop, converged, failed, confirm;
  int32_t prev_pass_had_cost;
  // pass totals of the last sweep (FusedPassOutput scalars)
  T pass_cost, pass_prev, pass_dual, pass_dx, pass_max_abs;
  int32_t pass_bad, pad0;
  // solve-loop scalars
  double last_cost, last_r_dual;
  double erg_mean;
  int64_t erg_count;
  double r_primal, dual_value, gap, fp_residual;
  double rep_r_primal, rep_r_dual, rep_gap, rep_objective;  // exact report
  int64_t trace_rows;
  int64_t gate_hits;
  // configuration (written once)
  int64_t max_iters, check_every, trace_every, trace_cap;
  double tol_primal, tol_dual, tol_gap, primal_scale;
  int32_t record_trace, relative;
  unsigned int ticket_merge, ticket_update, ticket_report, pad1;
  double jpart[4];  // sharded: replicated column-side partials of the update
  // fused-gate tail (tail.cu): the exact dual value and fixed-point terms of
  // an iteration are reduced one iteration later (or at finish) and patched
  int64_t pend_row;       // trace row awaiting its gap / fixed-point residual (-1: none)
  int32_t pend_valid;     // the tail's update partials of the last iteration are pending
  int32_t pend_use_dx;    // that iteration read C and wanted dx
  double pend_last_cost;  // last_cost seen by its gate
  double pend_dx;         // its pass dx^2
  double sum_p, sum_q;    // sum p_i, sum q_j (double, sequential; set at init)
  // cooperative tail: which of its two pending-partial buffers holds the
  // partials of pend_valid (tail.cu)
  int32_t pend_buf, pad_pm;
  // deferred bookkeeping of the cooperative tail (gate.cuh tail_decide /
  // tail_commit): what the last decided iteration still has to record
  int32_t cm_valid, cm_flags;  // flags: kCm* bits
  int64_t cm_k;                // the iteration (0-based) the record is of
  double cm_tot[5];            // pass totals {cost, prev, dual, dx, max|t|}
  double cm_r_primal, cm_r_dual, cm_gap, cm_dual, cm_last_cost;
};
constexpr int kCmCost = 1, kCmDual = 2, kCmFired = 4, kCmTrace = 8, kCmUseDx = 16, kCmFail = 32;

struct TraceRowDev {
  int64_t iter;
  double r_primal, r_dual, gap, objective, ergodic_objective,
      fixed_point_residual;
};

// Row-shard exchange over NVLink peer memory (tail.cu): every rank owns one
// exchange buffer, mapped by every peer (CUDA IPC across processes, plain
// device pointers within one):
//   [0, 256)          iteration flags: uint64 generation per sending rank
//   [256, 512)        setup-collective flags
//   [512, ...)        2 parity buffers x world slots of slot_bytes: slot s
//                     holds rank s's payload [v partial: n T, 16-B aligned |
//                     16 doubles of scalars]
//   [setup_off, ...)  2 parity buffers x world slots of setup_bytes
//   [off_ctr, ...)    the iteration tail's cross-rank counters: 2 parities x
//                     4 barriers, one 128-B line each (unsigned)
//   [off_acc, ...)    the exact accumulators (2 parities x kXaWords int64):
//                     every rank adds its row-side sums into every rank's
//   [off_vsum, ...)   the column sums, 2 parities x vwords x n int64: every
//                     rank adds its fixed-point column partials into every
//                     rank's (exact, so independent of the rank order)
// peers[r] = rank r's buffer as mapped here (peers[rank] = own buffer).
struct XArgs {
  char* const* peers;   // device array [world]
  int32_t world, rank;
  int64_t vec_bytes;    // round_up(n * sizeof(T), 16)
  int64_t slot_bytes;   // vec_bytes + 16 * 8
  int64_t buf_bytes;    // world * slot_bytes
  int64_t off_ctr, off_acc, off_vsum;
  int32_t vwords;       // int64 words per fixed-point column sum (1 fp32, 2 fp64)
  int32_t pad;
};
constexpr int64_t kXIterOff = 512;
constexpr int64_t kXSetupFlagOff = 256;

template <class T>
struct TailArgs {
  int64_t m, n, ld;
  int64_t m_global, n_global;  // problem sizes (rho, beta and inv_m/inv_n)
  int32_t folded_after;        // fold state of the array after this pass
  int32_t pad0;
  int64_t grid_cols;    // number of u strips
  int64_t grid_rows64;  // number of v strips (local)
  const T* ustrip;
  const T* vstrip;
  const PassPartial<T>* pass_partials;
  int64_t n_pass_partials;
  const T* p;
  const T* q;
  T* u;        // merged row sums (engine API)
  T* v;        // merged col sums
  T* r_new;
  T* s_new;
  const T* r_old;
  const T* s_old;
  T* phi;
  T* varphi;
  T* a;
  T* b;
  T rho;
  // pass properties
  int32_t reads_cost, want_dual, want_dx;
  int32_t solver;  // 0: engine pass only (no recursions)
  // reduction scratch
  double* dscratch;   // per-CTA double partials (update / report kernels)
  T* tscratch;        // per-CTA T partials (merge kernel)
  double* terms;      // exact mode per-element double terms (m+n)*3
  Book<T>* book;
  TraceRowDev* trace;
  // exact-mode per-tile scalar chains (tile order)
  const PassPartial<T>* tile_partials;
  int64_t n_tiles;
  // CUDA-graph IF node guarding the confirm report of this iteration
  unsigned long long cond;
  int32_t use_cond;
  // row-sharded multi-GPU (0: single device): merge/update/report write
  // their rank-local partials to these buffers for the NCCL allreduces
  int32_t sharded;
  T* pack;       // [v (n) | sum r, sum r^2, cost, prev, dual, dx, #bad]  (sum)
  T* pmax;       // [rank-local max|t|] (diagnostic, not reduced)
  double* dpack; // [dual_i, dphi^2, dphi, cross_i | obj, dual^2]    (sum)
  // cooperative tail (tail.cu): the arrays the confirm report streams
  const T* report_x;
  const T* report_c;
  unsigned long long* stamps;  // profiling aid: tail phase timestamps (or null)
  int32_t fused_gate;          // tail: gate on the algebraic dual value (one barrier less)
  int32_t tpar;                // tail: iteration parity (counter / pending-partial buffers)
  long long* ufx;              // fx: the sweep's fixed-point row / column sums (read + zeroed)
  long long* vfx;
  int32_t fx;
  int32_t pad_fx;
  double inv_n_d, inv_m_d;     // 1 / double(n_global), 1 / double(m_global)
  long long* xacc;             // exact accumulators, 2 parities x kXaWords
  // row shards (x.world > 1): the peers' buffers; the sweep's scalars land in
  // xloc (2 parities x kXaWords, this rank only) and are forwarded by the tail
  XArgs x;
  long long* xloc;
  int32_t pdl;                 // tail launched as a programmatic dependent of the sweep
  int32_t ctail;               // cluster tail allowed: max CTAs per cluster (0: grid tail)
};

// Cooperative per-iteration tail (tail.cu): merge + recursions + update +
// gate (+ confirm report) in one launch after K1 (fast order, one GPU).
// Its double partials use kTailDSlots words per CTA (tail.cu layout).
constexpr int kTailDSlots = 32;
template <class T>
int tail_grid(int device);
template <class T>
cudaError_t launch_tail(const TailArgs<T>& t, T* cpart, double* dpart, unsigned* bar, int grid,
                        cudaStream_t st);

// setup collective over the same buffers: out[i] = op_r in[r][i] in rank
// order (op 0 = sum, 1 = max); U in {float, double, int32}; one CTA
template <class U>
void launch_xallreduce(const U* in, U* out, int64_t count, int op, char* const* peers,
                       int world, int rank, int64_t setup_off, int64_t setup_bytes,
                       unsigned long long gen, cudaStream_t st);

// patch the pending exact dual value / fixed-point residual (end of a run)
template <class T>
void launch_tail_finalize(const TailArgs<T>& t, const double* dpart, int grid, cudaStream_t st);

// ---- kernel launchers (kernels.cu) ---------------------------------------
void launch_spin(unsigned long long ns, cudaStream_t st);
template <class T>
void launch_pass(const PassArgs<T>& a, int mode, bool want_dual, bool want_dx,
                 cudaStream_t st);
template <class T>
void launch_tile_chains(const PassArgs<T>& a, int mode, bool want_dual,
                        bool want_dx, int64_t bs, PassPartial<T>* tiles,
                        cudaStream_t st);
template <class T>
void launch_merge(const TailArgs<T>& t, bool exact, cudaStream_t st);
template <class T>
void launch_update(const TailArgs<T>& t, bool exact, cudaStream_t st);
template <class T>
void launch_report(const T* xy, const T* cost, const TailArgs<T>& t,
                   bool exact, bool always, cudaStream_t st);
template <class T>
void launch_finish(const TailArgs<T>& t, cudaStream_t st);
template <class T>
void launch_gate(const TailArgs<T>& t, cudaStream_t st);
template <class T>
void launch_report_final(const TailArgs<T>& t, bool always, cudaStream_t st);
template <class T>
void launch_init_sharded_finish(T* b, const T* q, int64_t n, const T* pack,
                                int64_t mn_global, Book<T>* book, cudaStream_t st);
template <class T>
void launch_init_x0(T* xy, const T* p, const T* q, int64_t m, int64_t n,
                    int64_t ld, cudaStream_t st);
template <class T>
void launch_init_sums(const T* xy, const T* p, const T* q, T* a, T* b,
                      int64_t m, int64_t n, int64_t ld, Book<T>* book,
                      cudaStream_t st, T* shard_pack = nullptr, bool x0_is_pq = false);
template <class T>
void launch_validate(const T* buf, int64_t m, int64_t n, int64_t ld,
                     unsigned long long* first_nonfinite,
                     unsigned long long* first_negative, cudaStream_t st);
template <class T>
void launch_materialize(const T* xy, const T* cost, T* out, T rho,
                        int folded, int64_t m, int64_t n, int64_t ld,
                        cudaStream_t st);
template <class T>
void launch_materialize_y(const T* xy, const T* cost, const T* phi, const T* varphi,
                          T* out, T rho, int folded, int64_t m, int64_t n, int64_t ld,
                          cudaStream_t st);

template <class T>
void launch_plan_max(const T* xy, const T* cost, T rho, int folded, int64_t m, int64_t n,
                     int64_t ld, unsigned long long* stats, cudaStream_t st);
template <class T>
void launch_plan_count(const T* xy, const T* cost, T rho, int folded, int64_t m, int64_t n,
                       int64_t ld, double thr, unsigned long long* stats, cudaStream_t st);

// residual_report / objective of an arbitrary (plan, cert) pair (report.cu);
// scratch: m + 3n doubles; out: r_primal, r_dual, gap, objective
template <class T>
void launch_residual_report(const T* x, const T* c, const T* mu, const T* nu, const T* p,
                            const T* q, int64_t m, int64_t n, bool exact, double* scratch,
                            double* out, cudaStream_t st);

// ---- K7 on-device problem generation (probgen.cu) -------------------------
void launch_gaussian_cmax(const double* xs, const double* xt, int64_t m, int64_t n,
                          unsigned long long* cmax_bits, cudaStream_t st);
template <class T>
void launch_gaussian_cost(const double* xs_local, const double* xt, int64_t m, int64_t n,
                          int64_t ld, const unsigned long long* cmax_bits, T* C,
                          cudaStream_t st);
template <class T>
void launch_uniform_cost(uint64_t seed, double lo, double hi, int64_t m, int64_t m_global,
                         int64_t row_begin, int64_t n, int64_t ld, T* C, cudaStream_t st);

int64_t kernel_launch_count();
void count_launch(int64_t k = 1);

inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

}  // namespace drotb
