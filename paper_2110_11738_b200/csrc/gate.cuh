// gate.cuh -- solve-loop scalar logic of the cooperative tails (tail.cu):
// Book copies through shared memory, the fused gate and the deferred exact
// dual / fixed-point patch.
#pragma once

#include "drotb_internal.hpp"
#include "sweep.cuh"

namespace drotb {

// The last CTA of a reduce-barrier runs the scalar logic (merge_scalars,
// gate_logic, report_decide -- one thread, many dependent reads of the Book)
// on a shared-memory copy: one coalesced round trip in, one out, instead of
// a global round trip per field (measured ~6 us per barrier otherwise).
template <class T>
__device__ __forceinline__ void book_load(Book<T>* dst, const Book<T>* src) {
  static_assert(sizeof(Book<T>) % 8 == 0, "Book is copied in 8-byte words");
  constexpr int W = static_cast<int>(sizeof(Book<T>) / 8);
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
  for (int k = threadIdx.x; k < W; k += blockDim.x) d[k] = __ldcg(s + k);
  __syncthreads();
}
template <class T>
__device__ __forceinline__ void book_store(Book<T>* dst, const Book<T>* src) {
  constexpr int W = static_cast<int>(sizeof(Book<T>) / 8);
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
  __syncthreads();
  for (int k = threadIdx.x; k < W; k += blockDim.x) d[k] = s[k];
  __syncthreads();
}

// Fused gate (t.fused_gate): the gate of iteration k runs right after the
// merge totals, on the dual value in closed form,
//   sum_i p_i phi_i^{k+1} = (sum p_i a_i - 2 sum p_i r_i + coef sum p_i) / n
// (and likewise for the columns), so the update phase needs no barrier
// behind it.  It is only the pre-filter of solver.hpp:474-504: the confirm
// report recomputes the exact dual value (sum of p_i * phi_i / rho, as the
// reference) and decides convergence.  The exact dual value and the
// fixed-point residual of an iteration (trace columns gap and
// fixed_point_residual) are reduced one iteration later -- or by the
// finalize kernel at the end of a run -- and patched into its trace row.
template <class T>
__device__ __forceinline__ void patch_pending(Book<T>* bk, TraceRowDev* trace, int64_t n_global,
                                              int64_t m_global, const double* d8,
                                              bool write_trace) {
  if (!bk->pend_valid) return;
  const double dual = d8[0] + d8[4];
  double fpr = __longlong_as_double(0x7ff8000000000000ULL);
  if (bk->record_trace) {  // rank-two identity (solver.hpp:443-472)
    double fp_sq = static_cast<double>(n_global) * d8[1] +
                   static_cast<double>(m_global) * d8[5] + 2.0 * d8[2] * d8[6];
    if (bk->pend_use_dx) fp_sq += bk->pend_dx + 2.0 * (d8[3] + d8[7]);
    fpr = sqrt(fmax(fp_sq, 0.0));
  }
  bk->dual_value = dual;
  bk->gap = fabs(bk->pend_last_cost - dual);
  bk->fp_residual = fpr;
  if (write_trace && trace && bk->pend_row >= 0 && bk->pend_row < bk->trace_cap) {
    TraceRowDev& row = trace[bk->pend_row];
    row.gap = bk->gap;
    row.fixed_point_residual = fpr;
  }
  bk->pend_valid = 0;
  bk->pend_row = -1;
}
template <class T>
__device__ __forceinline__ void patch_pending(Book<T>* bk, const TailArgs<T>& t,
                                              const double (&d8)[8], bool write_trace = true) {
  patch_pending<T>(bk, t.trace, t.n_global, t.m_global, d8, write_trace);
}

// ---- the fused-gate tail's scalar logic, split (tail.cu) --------------------
// tail_decide: what the next steps depend on -- the recursions' scalars, the
// stale residuals and the gate's control flow (merge_scalars + gate_fused,
// solver.hpp:266-289, 418-504) -- and a record of the rest; tail_commit:
// the rest (pass diagnostics, ergodic mean, result iteration count, the trace
// row, the pending-patch state), applied beside the NEXT iteration's decision
// (warp 1 of the next tail), by the confirm path, or by the finalize kernel.
// The decision reads nothing the commit writes, so the commit is off the
// critical path and the results are those of the sequential logic.
// tail_decide's inputs, in shared memory (the launch constants are set in
// the tail's prologue, off the critical path; the call passes two pointers)
template <class T>
struct DecideIn {
  T tot[8];                            // pass totals {cost, prev, dual, dx, max|t|, sum r, |r|^2, |s|^2}
  double sum_pa, sum_pr, sum_qb, sum_qs;  // exact merge sums
  double inv_n_d, inv_m_d;
  int64_t mn;                          // m_global + n_global
  T rho;
  int32_t totbad, folded_after, reads_cost, want_dual, want_dx;
};
template <class T>
__device__ __forceinline__ void decide_consts(DecideIn<T>* in, const TailArgs<T>& t) {
  in->inv_n_d = t.inv_n_d;
  in->inv_m_d = t.inv_m_d;
  in->mn = t.m_global + t.n_global;
  in->rho = t.rho;
  in->folded_after = t.folded_after;
  in->reads_cost = t.reads_cost;
  in->want_dual = t.want_dual;
  in->want_dx = t.want_dx;
}
template <class T>
__device__ __noinline__ void tail_decide(Book<T>* bk, const DecideIn<T>* in) {
  const T (&tot)[8] = in->tot;
  const int64_t k = bk->iter;
  bk->folded = in->folded_after;
  bk->cm_k = k;
#pragma unroll
  for (int q = 0; q < 5; ++q) bk->cm_tot[q] = static_cast<double>(tot[q]);
  bk->cm_valid = 1;
  if (in->totbad) {  // solver.hpp:266, 418-422
    bk->failed = 1;
    bk->stop = 1;
    bk->cm_flags = kCmFail;
    return;
  }
  const T beta = tot[5] / static_cast<T>(in->mn);
  bk->beta = beta;
  bk->coef = T(2) * beta - bk->alpha;
  bk->nr2 = tot[6];
  bk->ns2 = tot[7];
  const bool cost_valid = in->reads_cost != 0;
  const bool dual_valid = in->reads_cost && in->want_dual;
  if (cost_valid) bk->last_cost = static_cast<double>(tot[0]);
  if (dual_valid)
    bk->last_r_dual = sqrt(static_cast<double>(tot[2])) / static_cast<double>(in->rho);
  bk->alpha = bk->alpha - bk->beta;  // solver.hpp:289
  bk->iter = k + 1;
  const double dcoef = static_cast<double>(bk->coef);
  const double dual_alg = ((in->sum_pa - 2.0 * in->sum_pr + dcoef * bk->sum_p) * in->inv_n_d +
                           (in->sum_qb - 2.0 * in->sum_qs + dcoef * bk->sum_q) * in->inv_m_d) /
                          static_cast<double>(in->rho);
  const double r_primal = sqrt(static_cast<double>(bk->nr2) + static_cast<double>(bk->ns2));
  const double gap = fabs(bk->last_cost - dual_alg);
  const double gap_scale = bk->relative ? 1.0 / (1.0 + fabs(bk->last_cost)) : 1.0;
  const bool check = every(k + 1, bk->check_every);
  const bool trace_row = bk->record_trace && every(k + 1, bk->trace_every);
  // pre-filter with a slack above the closed form's rounding; gate_recheck
  // applies the reference's exact test before any confirm report
  const double slack = 1e-6 * bk->tol_gap + 1e-12 * fabs(bk->last_cost);
  const bool fire = check && r_primal * bk->primal_scale <= bk->tol_primal &&
                    bk->last_r_dual <= bk->tol_dual && gap * gap_scale <= bk->tol_gap + slack;
  if (fire)
    bk->confirm = 1;
  else if (k + 1 >= bk->max_iters)
    bk->stop = 1;
  bk->cm_flags = (cost_valid ? kCmCost : 0) | (dual_valid ? kCmDual : 0) |
                 (fire ? kCmFired : 0) | (trace_row ? kCmTrace : 0) |
                 ((in->reads_cost && in->want_dx) ? kCmUseDx : 0);
  bk->cm_r_primal = r_primal;
  bk->cm_r_dual = bk->last_r_dual;
  bk->cm_gap = gap;
  bk->cm_dual = dual_alg;
  bk->cm_last_cost = bk->last_cost;
}

// the commit record, copied before tail_decide of the next iteration
// overwrites it (the two run concurrently in the next tail)
struct CommitRec {
  int32_t valid, flags;
  int64_t k;
  double tot[5];
  double r_primal, r_dual, gap, dual, last_cost;
};
template <class T>
__device__ __forceinline__ CommitRec commit_snap(const Book<T>& b) {
  CommitRec c;
  c.valid = b.cm_valid;
  c.flags = b.cm_flags;
  c.k = b.cm_k;
#pragma unroll
  for (int q = 0; q < 5; ++q) c.tot[q] = b.cm_tot[q];
  c.r_primal = b.cm_r_primal;
  c.r_dual = b.cm_r_dual;
  c.gap = b.cm_gap;
  c.dual = b.cm_dual;
  c.last_cost = b.cm_last_cost;
  return c;
}

template <class T>
__device__ __forceinline__ void tail_commit(Book<T>* bk, TraceRowDev* trace, const CommitRec& c,
                                            bool write_trace) {
  if (!c.valid) return;
  bk->pass_cost = static_cast<T>(c.tot[0]);
  bk->pass_prev = static_cast<T>(c.tot[1]);
  bk->pass_dual = static_cast<T>(c.tot[2]);
  bk->pass_dx = static_cast<T>(c.tot[3]);
  bk->pass_max_abs = static_cast<T>(c.tot[4]);
  bk->pass_bad = (c.flags & kCmFail) ? 1 : 0;
  bk->iterations = c.k + 1;
  if (c.flags & kCmFail) return;
  const bool cost_valid = (c.flags & kCmCost) != 0;
  if (!bk->prev_pass_had_cost && cost_valid) erg_update(bk, c.tot[1]);
  if (cost_valid) erg_update(bk, c.tot[0]);
  bk->prev_pass_had_cost = cost_valid ? 1 : 0;
  const double nan = __longlong_as_double(0x7ff8000000000000ULL);
  bk->r_primal = c.r_primal;
  bk->dual_value = c.dual;
  bk->gap = c.gap;
  bk->fp_residual = nan;
  bk->pend_row = -1;
  if (c.flags & kCmTrace) {
    if (trace && bk->trace_rows < bk->trace_cap) {
      if (write_trace) {
        TraceRowDev& row = trace[bk->trace_rows];
        row.iter = c.k + 1;
        row.r_primal = c.r_primal;
        row.r_dual = c.r_dual;
        row.gap = c.gap;  // patched with the exact dual value later
        row.objective = c.last_cost;
        row.ergodic_objective = bk->erg_mean;
        row.fixed_point_residual = nan;  // patched later
      }
      bk->pend_row = bk->trace_rows;
    }
    bk->trace_rows += 1;
  }
  bk->pend_valid = 1;
  bk->pend_last_cost = c.last_cost;
  bk->pend_use_dx = (c.flags & kCmUseDx) ? 1 : 0;
  bk->pend_dx = c.tot[3];
  if (c.flags & kCmFired) bk->gate_hits += 1;
}
template <class T>
__device__ __forceinline__ void tail_commit(Book<T>* bk, const TailArgs<T>& t, const CommitRec& c,
                                            bool write_trace) {
  tail_commit<T>(bk, t.trace, c, write_trace);
}

// the previous iteration's commit + exact dual / fixed-point patch as one
// out-of-line call on shared-memory inputs (the cluster tail runs it once
// on a scratch Book to cache its code, then for real -- see tail.cu)
struct CommitIn {
  CommitRec c;
  double d8[8];
  TraceRowDev* trace;
  int64_t n_global, m_global;
  int32_t write_trace, pad;
};
template <class T>
__device__ __noinline__ void commit_patch(Book<T>* bk, const CommitIn* in) {
  tail_commit<T>(bk, in->trace, in->c, in->write_trace != 0);
  patch_pending<T>(bk, in->trace, in->n_global, in->m_global, in->d8, in->write_trace != 0);
}

// After patch_pending has put the EXACT dual value of the gated iteration in
// the Book: the reference's gap test on it (solver.hpp:498-504).  A pre-filter
// fire the exact gap rejects is withdrawn (no confirm report, the loop goes
// on -- or stops at max_iters, as the reference would).
template <class T>
__device__ void gate_recheck(Book<T>* bk) {
  if (!bk->confirm) return;
  const double gap_scale = bk->relative ? 1.0 / (1.0 + fabs(bk->pend_last_cost)) : 1.0;
  if (bk->gap * gap_scale <= bk->tol_gap) return;
  bk->confirm = 0;
  bk->gate_hits -= 1;
  bk->stop = bk->iter >= bk->max_iters ? 1 : 0;
}

}  // namespace drotb
