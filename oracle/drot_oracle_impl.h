/* drot_oracle_impl.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Type-generic body of the plain-C restatement of the reference DROT solver.
 * Included twice by drot_oracle.c with OT (float/double) and OSFX (f32/f64)
 * defined.  Every function names the reference lines it restates; the
 * arithmetic is written in the same association order (no FMA: the file is
 * compiled with -ffp-contract=off) so that it is bit-identical to the
 * reference in deterministic mode.
 */
#define OCAT2(a, b) a##_##b
#define OCAT(a, b) OCAT2(a, b)
#define OFN(name) OCAT(name, OSFX)

/* vec_sum / vec_norm_sq: matrix.hpp:99-104, 113-118 (ascending index). */
static OT OFN(vsum)(const OT* x, int64_t len) {
  OT acc = (OT)0;
  for (int64_t k = 0; k < len; ++k) acc += x[k];
  return acc;
}

static OT OFN(vnorm_sq)(const OT* x, int64_t len) {
  OT acc = (OT)0;
  for (int64_t k = 0; k < len; ++k) acc += x[k] * x[k];
  return acc;
}

/* One tiled sweep, FusedEngine<T>::run_pass (fused.hpp:206-357), in
 * deterministic mode (tile-ordered merge, fused.hpp:312-329).  Tiles follow
 * plan_tiles (tiles.cpp:20-47): bs x (ws*bs), ordered down each tile
 * column.  u_part / v_part are caller scratch of grid_cols*m and grid_rows*n. */
static void OFN(run_pass)(OT* xy, const OT* C, int64_t m, int64_t n,
                          const OT* phi, const OT* varphi, OT rho, int64_t bs,
                          int64_t ws, int fold_write, int input_folded,
                          int parity, int want_dual_opt, int want_dx_opt,
                          OT* row_sums, OT* col_sums, orc_pass_out* out) {
  const int reads_cost = !input_folded;
  const int want_dual = want_dual_opt && reads_cost;
  const int want_dx = want_dx_opt && !input_folded;
  const int want_prev = reads_cost && !input_folded;
  if (bs < 1) bs = 1;
  if (ws < 1) ws = 1;
  const int64_t tc = bs * ws;
  const int64_t grid_rows = (m + bs - 1) / bs;
  const int64_t grid_cols = (n + tc - 1) / tc;
  OT* u_part = (OT*)calloc((size_t)(grid_cols * m + 1), sizeof(OT));
  OT* v_part = (OT*)calloc((size_t)(grid_rows * n + 1), sizeof(OT));
  OT tot_cost = 0, tot_prev = 0, tot_dual = 0, tot_dx = 0, tot_max = 0;
  int tot_nonfinite = 0;

  for (int64_t gc = 0; gc < grid_cols; ++gc) {
    for (int64_t gr = 0; gr < grid_rows; ++gr) {
      const int64_t r0 = gr * bs, r1 = r0 + bs < m ? r0 + bs : m;
      const int64_t c0 = gc * tc, c1 = c0 + tc < n ? c0 + tc : n;
      OT* us = u_part + gc * m;
      OT* vs = v_part + gr * n;
      OT s_cost = 0, s_prev = 0, s_dual = 0, s_dx = 0, s_max = 0;
      int s_nonfinite = 0;
      for (int64_t i = r0; i < r1; ++i) us[i] = (OT)0;
      for (int64_t j = c0; j < c1; ++j) {
        OT* xc = xy + j * m;
        const OT* cc = C + j * m;
        const OT vj = varphi[j];
        OT colsum = (OT)0;
        for (int64_t i = r0; i < r1; ++i) {
          const OT x = xc[i];
          OT t, e = (OT)0, c = (OT)0;
          if (reads_cost) {
            c = cc[i];
            e = rho * c;
            if (parity == 0)
              t = ((x + phi[i]) + vj) - e;
            else
              t = ((x - e) + phi[i]) + vj;
          } else {
            t = (x + phi[i]) + vj;
          }
          const OT xp = t > (OT)0 ? t : (OT)0;
          xc[i] = fold_write ? xp - e : xp;
          us[i] += xp;
          colsum += xp;
          if (reads_cost) {
            s_cost += c * xp;
            if (want_prev) s_prev += c * x;
            if (want_dual) {
              const OT d = (phi[i] + vj) - e;
              if (d > (OT)0) s_dual += d * d;
            }
          }
          if (want_dx) {
            const OT dx = xp - x;
            s_dx += dx * dx;
          }
          const OT at = t < 0 ? -t : t;
          if (at > s_max) s_max = at;
          if (!isfinite((double)t)) s_nonfinite = 1;
        }
        vs[j] = colsum;
      }
      /* merge in tile order, fused.hpp:322-329 */
      tot_cost += s_cost;
      tot_prev += s_prev;
      tot_dual += s_dual;
      tot_dx += s_dx;
      if (s_max > tot_max) tot_max = s_max;
      tot_nonfinite = tot_nonfinite || s_nonfinite;
    }
  }
  for (int64_t i = 0; i < m; ++i) row_sums[i] = (OT)0;
  for (int64_t j = 0; j < n; ++j) col_sums[j] = (OT)0;
  for (int64_t gc = 0; gc < grid_cols; ++gc)
    for (int64_t i = 0; i < m; ++i) row_sums[i] += u_part[gc * m + i];
  for (int64_t gr = 0; gr < grid_rows; ++gr)
    for (int64_t j = 0; j < n; ++j) col_sums[j] += v_part[gr * n + j];
  free(u_part);
  free(v_part);

  out->cost_dot = (double)tot_cost;
  out->cost_valid = reads_cost;
  out->max_abs = (double)tot_max;
  out->nonfinite = tot_nonfinite;
  out->dual_sq = (double)tot_dual;
  out->dual_valid = want_dual;
  out->dx_sq = (double)tot_dx;
  out->dx_valid = want_dx;
  out->prev_cost_dot = (double)tot_prev;
  out->prev_cost_valid = want_prev;
}

/* Public pass entry: fused_pass (fused.hpp:127-134), fused_pass_skip_cost
 * (:140-155, including the fold_state_mismatch guard :146-149) and
 * unfused_pass (:359-531; bitwise equal to the fused pass in deterministic
 * mode, test_fused.cpp:123-137, so only its traffic accounting differs). */
int OFN(orc_pass)(OT* xy, const OT* C, int64_t m, int64_t n, const OT* phi,
                  const OT* varphi, OT rho, int64_t bs, int64_t ws,
                  int32_t kind, int32_t fold, int32_t* folded_inout,
                  int32_t parity, int32_t want_dual, int32_t want_dx,
                  OT* row_sums, OT* col_sums, orc_pass_out* out,
                  orc_counters* counters) {
  orc_pass_out tmp;
  if (!out) out = &tmp;
  const uint64_t cells = (uint64_t)(m * n);
  if (kind == ORC_PASS_SKIP_COST) {
    if ((fold != 0) == (*folded_inout != 0)) return 1 + ORC_ERRC_FOLD_STATE_MISMATCH;
    OFN(run_pass)(xy, C, m, n, phi, varphi, rho, bs, ws, fold != 0, !fold,
                  fold ? 0 : 1, want_dual, want_dx, row_sums, col_sums, out);
    *folded_inout = fold ? 1 : 0;
    if (counters) {
      counters->passes += 1;
      counters->xy_elems_read += cells;
      counters->xy_elems_written += cells;
      if (fold) counters->cost_elems_read += cells;
    }
  } else if (kind == ORC_PASS_UNFUSED) {
    OFN(run_pass)(xy, C, m, n, phi, varphi, rho, bs, ws, 0, 0, parity,
                  want_dual, want_dx, row_sums, col_sums, out);
    out->prev_cost_valid = 1;
    if (counters) {
      counters->passes += 1;
      counters->xy_elems_read += 4 * cells;
      counters->xy_elems_written += cells;
      counters->cost_elems_read += 2 * cells;
    }
  } else {
    OFN(run_pass)(xy, C, m, n, phi, varphi, rho, bs, ws, 0, 0, parity,
                  want_dual, want_dx, row_sums, col_sums, out);
    if (counters) {
      counters->passes += 1;
      counters->xy_elems_read += cells;
      counters->xy_elems_written += cells;
      counters->cost_elems_read += cells;
    }
  }
  return 0;
}

/* check_problem / check_marginal: problem.hpp:103-136. */
static int OFN(check_marginal)(const OT* v, int64_t len, double tol) {
  if (len == 0) return 1 + ORC_ERRC_EMPTY_DIMENSION;
  double sum = 0;
  for (int64_t k = 0; k < len; ++k) {
    if (!isfinite((double)v[k])) return 1 + ORC_ERRC_NON_FINITE_ENTRY;
    if (v[k] < (OT)0) return 1 + ORC_ERRC_MARGINAL_NOT_SIMPLEX;
    sum += (double)v[k];
  }
  if (fabs(sum - 1.0) > tol) return 1 + ORC_ERRC_MARGINAL_NOT_SIMPLEX;
  return 0;
}

int OFN(orc_check_problem)(const OT* C, int64_t m, int64_t n, const OT* p,
                           const OT* q) {
  if (m == 0 || n == 0) return 1 + ORC_ERRC_EMPTY_DIMENSION;
  for (int64_t k = 0; k < m * n; ++k) {
    if (!isfinite((double)C[k])) return 1 + ORC_ERRC_NON_FINITE_ENTRY;
    if (C[k] < (OT)0) return 1 + ORC_ERRC_NEGATIVE_COST;
  }
  int rc = OFN(check_marginal)(p, m, 1e-12);
  if (rc) return rc;
  return OFN(check_marginal)(q, n, 1e-12);
}

/* DrotState<T> (solver.hpp:98-114). */
typedef struct {
  OT* xy;
  int folded;
  OT *phi, *varphi, *a, *b, *r, *s;
  OT alpha, beta;
  int64_t iter;
} OFN(state);

static void OFN(state_free)(OFN(state) * st) {
  free(st->xy);
  free(st->phi);
  free(st->varphi);
  free(st->a);
  free(st->b);
  free(st->r);
  free(st->s);
}

/* init_state: solver.hpp:143-186.  row_sums/col_sums of X0 are the untiled
 * sequential matrix.hpp:128-149 reductions. */
static int OFN(init_state)(OFN(state) * st, const OT* C, int64_t m, int64_t n,
                           const OT* p, const OT* q, const OT* x0) {
  (void)C;
  memset(st, 0, sizeof(*st));
  st->xy = (OT*)malloc(sizeof(OT) * (size_t)(m * n));
  if (x0) {
    for (int64_t k = 0; k < m * n; ++k)
      if (!(x0[k] >= (OT)0) || !isfinite((double)x0[k])) {
        free(st->xy);
        st->xy = NULL;
        return 1 + ORC_ERRC_INVALID_INITIAL_PLAN;
      }
    memcpy(st->xy, x0, sizeof(OT) * (size_t)(m * n));
  } else {
    for (int64_t j = 0; j < n; ++j) {
      const OT qj = q[j];
      for (int64_t i = 0; i < m; ++i) st->xy[j * m + i] = p[i] * qj;
    }
  }
  st->folded = 0;
  st->phi = (OT*)calloc((size_t)m, sizeof(OT));
  st->varphi = (OT*)calloc((size_t)n, sizeof(OT));
  st->a = (OT*)calloc((size_t)m, sizeof(OT));
  st->b = (OT*)calloc((size_t)n, sizeof(OT));
  st->r = (OT*)malloc(sizeof(OT) * (size_t)m);
  st->s = (OT*)malloc(sizeof(OT) * (size_t)n);
  for (int64_t j = 0; j < n; ++j) {
    const OT* col = st->xy + j * m;
    for (int64_t i = 0; i < m; ++i) st->a[i] += col[i];
  }
  for (int64_t i = 0; i < m; ++i) st->a[i] -= p[i];
  for (int64_t j = 0; j < n; ++j) {
    const OT* col = st->xy + j * m;
    OT acc = (OT)0;
    for (int64_t i = 0; i < m; ++i) acc += col[i];
    st->b[j] = acc;
  }
  for (int64_t j = 0; j < n; ++j) st->b[j] -= q[j];
  st->alpha = OFN(vsum)(st->a, m) / (OT)(m + n);
  memcpy(st->r, st->a, sizeof(OT) * (size_t)m);
  memcpy(st->s, st->b, sizeof(OT) * (size_t)n);
  st->beta = st->alpha;
  st->iter = 0;
  return 0;
}

/* detail::step_impl: solver.hpp:238-307. */
static int OFN(step_impl)(OFN(state) * st, const OT* C, int64_t m, int64_t n,
                          const OT* p, const OT* q, OT rho,
                          const orc_config* cfg, int want_dual, int want_dx,
                          OT* u, OT* v, orc_pass_out* out) {
  const int parity = (int)(st->iter & 1);
  if (cfg->engine == 0) {
    if (st->folded) return 1 + ORC_ERRC_FOLD_STATE_MISMATCH;
    OFN(run_pass)(st->xy, C, m, n, st->phi, st->varphi, rho, cfg->block_rows,
                  cfg->work_size, 0, 0, parity, want_dual, want_dx, u, v, out);
    out->prev_cost_valid = 1;
  } else if (cfg->skip_cost) {
    const int fold = !st->folded;
    OFN(run_pass)(st->xy, C, m, n, st->phi, st->varphi, rho, cfg->block_rows,
                  cfg->work_size, fold, !fold, fold ? 0 : 1, want_dual,
                  want_dx, u, v, out);
    st->folded = fold;
  } else {
    OFN(run_pass)(st->xy, C, m, n, st->phi, st->varphi, rho, cfg->block_rows,
                  cfg->work_size, 0, 0, parity, want_dual, want_dx, u, v, out);
  }
  if (out->nonfinite) return 0;

  for (int64_t i = 0; i < m; ++i) st->r[i] = u[i] - p[i];
  for (int64_t j = 0; j < n; ++j) st->s[j] = v[j] - q[j];
  const OT beta = OFN(vsum)(st->r, m) / (OT)(m + n);
  st->beta = beta;
  const OT coef = (OT)2 * beta - st->alpha;
  const OT inv_n = (OT)1 / (OT)n;
  const OT inv_m = (OT)1 / (OT)m;
  for (int64_t i = 0; i < m; ++i)
    st->phi[i] = (st->a[i] - (OT)2 * st->r[i] + coef) * inv_n;
  for (int64_t j = 0; j < n; ++j)
    st->varphi[j] = (st->b[j] - (OT)2 * st->s[j] + coef) * inv_m;
  for (int64_t i = 0; i < m; ++i) st->a[i] -= st->r[i];
  for (int64_t j = 0; j < n; ++j) st->b[j] -= st->s[j];
  st->alpha -= beta;
  st->iter += 1;
  return 0;
}

/* detail::state_report: solver.hpp:312-354 (double accumulation, unfold on
 * the fly when the array is folded). */
static void OFN(state_report)(const OFN(state) * st, const OT* C, int64_t m,
                              int64_t n, const OT* p, const OT* q, OT rho,
                              orc_report* rep) {
  double obj = 0, dual_sq = 0;
  for (int64_t j = 0; j < n; ++j) {
    const OT* xc = st->xy + j * m;
    const OT* cc = C + j * m;
    const double nu_j = (double)st->varphi[j] / rho;
    for (int64_t i = 0; i < m; ++i) {
      const double c = (double)cc[i];
      double x = (double)xc[i];
      if (st->folded) {
        x += (double)rho * c;
        if (x < 0) x = 0;
      }
      obj += c * x;
      const double slack = (double)st->phi[i] / rho + nu_j - c;
      if (slack > 0) dual_sq += slack * slack;
    }
  }
  double dual_value = 0;
  for (int64_t i = 0; i < m; ++i)
    dual_value += (double)p[i] * (double)st->phi[i] / rho;
  for (int64_t j = 0; j < n; ++j)
    dual_value += (double)q[j] * (double)st->varphi[j] / rho;
  rep->objective = obj;
  rep->r_primal = sqrt((double)OFN(vnorm_sq)(st->r, m) +
                       (double)OFN(vnorm_sq)(st->s, n));
  rep->r_dual = sqrt(dual_sq);
  rep->gap = fabs(obj - dual_value);
}

/* DrotConfig::resolved_rho: solver.hpp:77-83. */
static int OFN(resolved_rho)(const orc_config* cfg, int64_t m, int64_t n,
                             double* rho) {
  const double r = cfg->has_rho_override ? cfg->rho_override
                                         : cfg->rho0 / (double)(m + n);
  if (!(r > 0) || !isfinite(r)) return 1 + ORC_ERRC_NON_POSITIVE_RHO;
  *rho = r;
  return 0;
}

/* drot::solve<T>: solver.hpp:372-540. */
int OFN(orc_solve)(const OT* C, int64_t m, int64_t n, const OT* p,
                   const OT* q, const orc_config* cfg, const OT* x0, OT* plan,
                   OT* mu, OT* nu, orc_report* rep_out, orc_trace_row* trace,
                   int64_t trace_cap, int64_t* trace_len, int64_t* iters_out,
                   int32_t* status_out, double* wall) {
  int rc = OFN(orc_check_problem)(C, m, n, p, q);
  if (rc) return rc;
  double rho_d;
  rc = OFN(resolved_rho)(cfg, m, n, &rho_d);
  if (rc) return rc;
  const OT rho = (OT)rho_d;
  OFN(state) st;
  rc = OFN(init_state)(&st, C, m, n, p, q, x0);
  if (rc) return rc;

  const double p_norm = sqrt((double)OFN(vnorm_sq)(p, m));
  const double q_norm = sqrt((double)OFN(vnorm_sq)(q, n));
  const double primal_scale =
      cfg->relative_tolerances ? 1.0 / (1.0 + p_norm + q_norm) : 1.0;

  int status = ORC_MAX_ITERS;
  double erg_mean = 0;
  int64_t erg_count = 0;
  const int want_fp = cfg->record_trace != 0;
  OT* prev_phi = (OT*)malloc(sizeof(OT) * (size_t)m);
  OT* prev_varphi = (OT*)malloc(sizeof(OT) * (size_t)n);
  OT* prev_r = (OT*)malloc(sizeof(OT) * (size_t)m);
  OT* prev_s = (OT*)malloc(sizeof(OT) * (size_t)n);
  OT* u = (OT*)malloc(sizeof(OT) * (size_t)m);
  OT* v = (OT*)malloc(sizeof(OT) * (size_t)n);
  double last_cost = NAN;
  double last_r_dual = INFINITY;
  int prev_pass_had_cost = 1;
  int failed = 0;
  int64_t iterations = 0, rows = 0;
  orc_report rep = {0, 0, 0, 0};

  for (int64_t k = 0; k < cfg->max_iters; ++k) {
    if (want_fp) {
      memcpy(prev_phi, st.phi, sizeof(OT) * (size_t)m);
      memcpy(prev_varphi, st.varphi, sizeof(OT) * (size_t)n);
      memcpy(prev_r, st.r, sizeof(OT) * (size_t)m);
      memcpy(prev_s, st.s, sizeof(OT) * (size_t)n);
    }
    orc_pass_out out;
    rc = OFN(step_impl)(&st, C, m, n, p, q, rho, cfg, 1, want_fp, u, v, &out);
    if (rc) break;
    iterations = k + 1;
    if (out.nonfinite) {
      failed = 1;
      break;
    }
    if (!prev_pass_had_cost && out.prev_cost_valid) {
      ++erg_count;
      erg_mean += (out.prev_cost_dot - erg_mean) / (double)erg_count;
    }
    if (out.cost_valid) {
      last_cost = out.cost_dot;
      ++erg_count;
      erg_mean += (last_cost - erg_mean) / (double)erg_count;
    }
    prev_pass_had_cost = out.cost_valid;
    if (out.dual_valid) last_r_dual = sqrt(out.dual_sq) / (double)rho;

    const int check = ((k + 1) % cfg->check_every) == 0;
    const int trace_row = cfg->record_trace && ((k + 1) % cfg->trace_every) == 0;

    double fp_residual = NAN;
    if (want_fp) {
      double dphi_sq = 0, dvarphi_sq = 0, sum_dphi = 0, sum_dvarphi = 0,
             cross = 0;
      for (int64_t i = 0; i < m; ++i) {
        const double d = (double)st.phi[i] - (double)prev_phi[i];
        dphi_sq += d * d;
        sum_dphi += d;
        cross += d * ((double)st.r[i] - (double)prev_r[i]);
      }
      for (int64_t j = 0; j < n; ++j) {
        const double d = (double)st.varphi[j] - (double)prev_varphi[j];
        dvarphi_sq += d * d;
        sum_dvarphi += d;
        cross += d * ((double)st.s[j] - (double)prev_s[j]);
      }
      double fp_sq = (double)n * dphi_sq + (double)m * dvarphi_sq +
                     2.0 * sum_dphi * sum_dvarphi;
      if (out.dx_valid) fp_sq += out.dx_sq + 2.0 * cross;
      fp_residual = sqrt(fp_sq > 0.0 ? fp_sq : 0.0);
    }

    if (check || trace_row) {
      const double r_primal = sqrt((double)OFN(vnorm_sq)(st.r, m) +
                                   (double)OFN(vnorm_sq)(st.s, n));
      double dual_value = 0;
      for (int64_t i = 0; i < m; ++i)
        dual_value += (double)p[i] * (double)st.phi[i] / (double)rho;
      for (int64_t j = 0; j < n; ++j)
        dual_value += (double)q[j] * (double)st.varphi[j] / (double)rho;
      const double gap = fabs(last_cost - dual_value);
      const double gap_scale =
          cfg->relative_tolerances ? 1.0 / (1.0 + fabs(last_cost)) : 1.0;
      if (trace_row) {
        if (trace && rows < trace_cap) {
          orc_trace_row* tr = &trace[rows];
          tr->iter = k + 1;
          tr->r_primal = r_primal;
          tr->r_dual = last_r_dual;
          tr->gap = gap;
          tr->objective = last_cost;
          tr->ergodic_objective = erg_mean;
          tr->fixed_point_residual = fp_residual;
        }
        ++rows;
      }
      if (check && r_primal * primal_scale <= cfg->tol_primal &&
          last_r_dual <= cfg->tol_dual && gap * gap_scale <= cfg->tol_gap) {
        orc_report exact;
        OFN(state_report)(&st, C, m, n, p, q, rho, &exact);
        const double egs = cfg->relative_tolerances
                               ? 1.0 / (1.0 + fabs(exact.objective))
                               : 1.0;
        if (exact.r_primal * primal_scale <= cfg->tol_primal &&
            exact.r_dual <= cfg->tol_dual &&
            exact.gap * egs <= cfg->tol_gap) {
          status = ORC_CONVERGED;
          rep = exact;
          break;
        }
      }
    }
  }
  if (wall) *wall = 0;
  if (rc == 0) {
    if (failed) status = ORC_NUMERICAL_FAILURE;
    /* materialize_plan: solver.hpp:204-217 */
    if (plan) {
      for (int64_t k = 0; k < m * n; ++k) {
        if (st.folded) {
          const OT val = st.xy[k] + rho * C[k];
          plan[k] = val > (OT)0 ? val : (OT)0;
        } else {
          plan[k] = st.xy[k];
        }
      }
    }
    /* recover_duals: solver.hpp:188-199 */
    if (mu)
      for (int64_t i = 0; i < m; ++i) mu[i] = st.phi[i] / rho;
    if (nu)
      for (int64_t j = 0; j < n; ++j) nu[j] = st.varphi[j] / rho;
    if (status != ORC_CONVERGED && !failed)
      OFN(state_report)(&st, C, m, n, p, q, rho, &rep);
    if (failed) rep.r_primal = rep.r_dual = rep.gap = rep.objective = NAN;
    if (rep_out) *rep_out = rep;
    if (trace_len) *trace_len = rows;
    if (iters_out) *iters_out = iterations;
    if (status_out) *status_out = status;
  }
  free(prev_phi);
  free(prev_varphi);
  free(prev_r);
  free(prev_s);
  free(u);
  free(v);
  OFN(state_free)(&st);
  return rc;
}

/* init_state + k x drot_step (solver.hpp:361-370: default PassOptions, i.e.
 * want_dual = want_dx = false; non-finite -> non_finite_iterate), then the
 * raw state and detail::state_report. */
int OFN(orc_steps)(const OT* C, int64_t m, int64_t n, const OT* p, const OT* q,
                   const orc_config* cfg, int64_t k, OT* xy, int32_t* folded,
                   OT* phi, OT* varphi, OT* a, OT* b, OT* alpha, OT* r, OT* s,
                   OT* beta, orc_report* rep) {
  double rho_d;
  int rc = OFN(resolved_rho)(cfg, m, n, &rho_d);
  if (rc) return rc;
  const OT rho = (OT)rho_d;
  OFN(state) st;
  rc = OFN(init_state)(&st, C, m, n, p, q, NULL);
  if (rc) return rc;
  OT* u = (OT*)malloc(sizeof(OT) * (size_t)m);
  OT* v = (OT*)malloc(sizeof(OT) * (size_t)n);
  for (int64_t it = 0; it < k && rc == 0; ++it) {
    orc_pass_out out;
    rc = OFN(step_impl)(&st, C, m, n, p, q, rho, cfg, 0, 0, u, v, &out);
    if (rc == 0 && out.nonfinite) rc = 1 + ORC_ERRC_NON_FINITE_ITERATE;
  }
  if (rc == 0) {
    if (xy) memcpy(xy, st.xy, sizeof(OT) * (size_t)(m * n));
    if (folded) *folded = st.folded;
    if (phi) memcpy(phi, st.phi, sizeof(OT) * (size_t)m);
    if (varphi) memcpy(varphi, st.varphi, sizeof(OT) * (size_t)n);
    if (a) memcpy(a, st.a, sizeof(OT) * (size_t)m);
    if (b) memcpy(b, st.b, sizeof(OT) * (size_t)n);
    if (alpha) *alpha = st.alpha;
    if (r) memcpy(r, st.r, sizeof(OT) * (size_t)m);
    if (s) memcpy(s, st.s, sizeof(OT) * (size_t)n);
    if (beta) *beta = st.beta;
    if (rep) OFN(state_report)(&st, C, m, n, p, q, rho, rep);
  }
  free(u);
  free(v);
  OFN(state_free)(&st);
  return rc;
}

/* residual_report: problem.hpp:174-225. */
int OFN(orc_residual_report)(const OT* C, int64_t m, int64_t n, const OT* p,
                             const OT* q, const OT* plan, const OT* mu,
                             const OT* nu, orc_report* rep) {
  double* row = (double*)calloc((size_t)m, sizeof(double));
  double obj = 0, dual_sq = 0, col_sq = 0;
  for (int64_t j = 0; j < n; ++j) {
    const OT* xc = plan + j * m;
    const OT* cc = C + j * m;
    const double nu_j = (double)nu[j];
    double colsum = 0;
    for (int64_t i = 0; i < m; ++i) {
      const double x = (double)xc[i];
      const double c = (double)cc[i];
      colsum += x;
      row[i] += x;
      obj += c * x;
      const double slack = (double)mu[i] + nu_j - c;
      if (slack > 0) dual_sq += slack * slack;
    }
    const double cd = colsum - (double)q[j];
    col_sq += cd * cd;
  }
  double row_sq = 0;
  for (int64_t i = 0; i < m; ++i) {
    const double rd = row[i] - (double)p[i];
    row_sq += rd * rd;
  }
  double dual_value = 0;
  for (int64_t i = 0; i < m; ++i) dual_value += (double)p[i] * (double)mu[i];
  for (int64_t j = 0; j < n; ++j) dual_value += (double)q[j] * (double)nu[j];
  free(row);
  rep->objective = obj;
  rep->r_primal = sqrt(row_sq + col_sq);
  rep->r_dual = sqrt(dual_sq);
  rep->gap = fabs(obj - dual_value);
  return 0;
}

#undef OFN
#undef OCAT
#undef OCAT2
