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
__device__ void patch_pending(Book<T>* bk, const TailArgs<T>& t, const double (&d8)[8],
                              bool write_trace = true) {
  if (!bk->pend_valid) return;
  const double dual = d8[0] + d8[4];
  double fpr = __longlong_as_double(0x7ff8000000000000ULL);
  if (bk->record_trace) {  // rank-two identity (solver.hpp:443-472)
    double fp_sq = static_cast<double>(t.n_global) * d8[1] +
                   static_cast<double>(t.m_global) * d8[5] + 2.0 * d8[2] * d8[6];
    if (bk->pend_use_dx) fp_sq += bk->pend_dx + 2.0 * (d8[3] + d8[7]);
    fpr = sqrt(fmax(fp_sq, 0.0));
  }
  bk->dual_value = dual;
  bk->gap = fabs(bk->pend_last_cost - dual);
  bk->fp_residual = fpr;
  if (write_trace && t.trace && bk->pend_row >= 0 && bk->pend_row < bk->trace_cap) {
    TraceRowDev& row = t.trace[bk->pend_row];
    row.gap = bk->gap;
    row.fixed_point_residual = fpr;
  }
  bk->pend_valid = 0;
  bk->pend_row = -1;
}

template <class T>
__device__ void gate_fused(Book<T>* bk, const TailArgs<T>& t, double dual_alg,
                           bool write_trace = true) {
  bk->alpha = bk->alpha - bk->beta;  // solver.hpp:289
  const int64_t k = bk->iter;
  bk->iter = k + 1;
  const double nan = __longlong_as_double(0x7ff8000000000000ULL);
  const double r_primal = sqrt(static_cast<double>(bk->nr2) + static_cast<double>(bk->ns2));
  const double gap = fabs(bk->last_cost - dual_alg);
  const double gap_scale = bk->relative ? 1.0 / (1.0 + fabs(bk->last_cost)) : 1.0;
  bk->r_primal = r_primal;
  bk->dual_value = dual_alg;
  bk->gap = gap;
  bk->fp_residual = nan;
  const bool check = every(k + 1, bk->check_every);
  const bool trace_row = bk->record_trace && every(k + 1, bk->trace_every);
  bk->pend_row = -1;
  if (trace_row) {
    if (t.trace && bk->trace_rows < bk->trace_cap) {
      if (write_trace) {
        TraceRowDev& row = t.trace[bk->trace_rows];
        row.iter = k + 1;
        row.r_primal = r_primal;
        row.r_dual = bk->last_r_dual;
        row.gap = gap;  // patched with the exact dual value later
        row.objective = bk->last_cost;
        row.ergodic_objective = bk->erg_mean;
        row.fixed_point_residual = nan;  // patched later
      }
      bk->pend_row = bk->trace_rows;
    }
    bk->trace_rows += 1;
  }
  bk->pend_valid = 1;
  bk->pend_last_cost = bk->last_cost;
  bk->pend_use_dx = (t.reads_cost && t.want_dx) ? 1 : 0;
  bk->pend_dx = static_cast<double>(bk->pass_dx);
  // pre-filter: the closed-form dual value differs from the reference's sum
  // by rounding only, so the gap test gets a slack far above that rounding
  // (and far below tol_gap); gate_recheck then applies the reference's exact
  // test (solver.hpp:498-504) before any confirm report runs
  const double slack = 1e-6 * bk->tol_gap + 1e-12 * fabs(bk->last_cost);
  const bool fire = check && r_primal * bk->primal_scale <= bk->tol_primal &&
                    bk->last_r_dual <= bk->tol_dual && gap * gap_scale <= bk->tol_gap + slack;
  if (fire) {
    bk->confirm = 1;
    bk->gate_hits += 1;
  } else if (k + 1 >= bk->max_iters) {
    bk->stop = 1;
  }
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
