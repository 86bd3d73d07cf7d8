/* oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Shared declarations for the two CPU oracles under oracle/:
 *   - ref_*  : the UNMODIFIED reference (/root/reference/proj/core) compiled
 *              from its own sources into oracle/_ref/libdrotref.so by
 *              oracle/Makefile, wrapped by oracle/ref_shim.cpp;
 *   - orc_*  : oracle/drot_oracle.c, a plain-C restatement of the reference
 *              algorithm (each function cites the reference file:line).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries, and only as the checker or
 * as the timed CPU baseline.  The product (paper_2110_11738_b200/) never links
 * or calls anything declared here.
 */
#ifndef DROT_ORACLE_H_
#define DROT_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors drot::DrotConfig (solver.hpp:51-88). */
typedef struct orc_config {
  double rho0;
  int32_t has_rho_override;
  int32_t relative_tolerances;
  double rho_override;
  double tol_primal, tol_dual, tol_gap;
  int64_t max_iters, check_every;
  int32_t engine;        /* 0 = reference (unfused), 1 = fused */
  int32_t skip_cost;
  int32_t deterministic;
  int32_t record_trace;
  int64_t workers, block_rows, work_size;
  int64_t trace_every;
} orc_config;

/* Mirrors drot::ResidualReport (problem.hpp:57-62). */
typedef struct orc_report {
  double r_primal, r_dual, gap, objective;
} orc_report;

/* Mirrors drot::TraceRow (problem.hpp:77-85). */
typedef struct orc_trace_row {
  int64_t iter;
  double r_primal, r_dual, gap, objective, ergodic_objective,
      fixed_point_residual;
} orc_trace_row;

/* Scalars of drot::FusedPassOutput (fused.hpp:42-60); T values widened to
 * double (exact for float). */
typedef struct orc_pass_out {
  double cost_dot, max_abs, dual_sq, dx_sq, prev_cost_dot;
  int32_t cost_valid, nonfinite, dual_valid, dx_valid, prev_cost_valid;
  int32_t pad_;
} orc_pass_out;

/* Mirrors drot::MemoryCounters (fused.hpp:34-39). */
typedef struct orc_counters {
  uint64_t passes, xy_elems_read, xy_elems_written, cost_elems_read;
} orc_counters;

/* Status codes: drot::SolveStatus (problem.hpp:66). */
enum { ORC_CONVERGED = 0, ORC_MAX_ITERS = 1, ORC_NUMERICAL_FAILURE = 2 };

/* Pass kinds. */
enum { ORC_PASS_FUSED = 0, ORC_PASS_SKIP_COST = 1, ORC_PASS_UNFUSED = 2 };

/* Return convention for every entry point: 0 on success, otherwise
 * 1 + ordinal of drot::Errc (errors.hpp:24-46). */

#ifdef __cplusplus
}
#endif

#endif /* DROT_ORACLE_H_ */
