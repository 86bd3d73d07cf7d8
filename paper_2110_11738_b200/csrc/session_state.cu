// session_state.cu -- the reference's external-state entry points on a
// Session<T>: drot_step on caller-owned DrotState (solver.hpp:361-370) and
// the FusedEngine pass API (fused.hpp:107-202).
#include "session.hpp"

namespace drotb {


// ---- external-state single step (drot_step, solver.hpp:361-370) --------
template <class T>
int Session<T>::load_state(const T* xy, int32_t folded, const T* rs, const T* cs, const T* ya, const T* yb, T alpha, const T* r, const T* s, T beta, int64_t iter) {
  RC_TRY(resolve_rho());
  if (tbar) CUDA_TRY(cudaMemsetAsync(tbar, 0, 1024 * sizeof(unsigned), stream));  // tail counters
  if (fx) {  // an external state carries no bound on its row sums: strips
    drop_graphs();
    fx = false;
  }
  if (xacc) CUDA_TRY(cudaMemsetAsync(xacc, 0, sizeof(long long) * 2 * kXaWords, stream));
  RC_TRY(upload_matrix(X, xy, false));
  CUDA_TRY(cudaMemcpyAsync(phi, rs, sizeof(T) * m, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(varphi, cs, sizeof(T) * n, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(a, ya, sizeof(T) * m, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(b, yb, sizeof(T) * n, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(rb[iter & 1], r, sizeof(T) * m, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(sb[iter & 1], s, sizeof(T) * n, cudaMemcpyHostToDevice, stream));
  Book<T> hb;
  std::memset(&hb, 0, sizeof(hb));
  hb.alpha = alpha;
  hb.beta = beta;
  hb.iter = iter;
  hb.folded = folded;
  hb.last_cost = std::numeric_limits<double>::quiet_NaN();
  hb.last_r_dual = std::numeric_limits<double>::infinity();
  hb.prev_pass_had_cost = 1;
  hb.max_iters = std::numeric_limits<int64_t>::max();
  hb.check_every = 1;
  hb.trace_every = 1;
  hb.tol_primal = hb.tol_dual = hb.tol_gap = -1.0;
  hb.pend_row = -1;
  hb.pend_buf = 0;
  CUDA_TRY(cudaMemcpyAsync(book, &hb, sizeof(hb), cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  want_dual = false;  // default PassOptions (solver.hpp:367)
  want_dx = false;
  gate = false;
  h_iter = iter;
  h_folded = folded != 0;
  initialized = true;
  return 0;
}


template <class T>
int Session<T>::store_state(T* xy, int32_t* folded, T* rs, T* cs, T* ya, T* yb, T* alpha, T* r, T* s, T* beta, int64_t* iter, bool full) {
  RC_TRY(finalize_pending());
  Book<T> hb;
  RC_TRY(read_book(&hb));
  RC_TRY(download_matrix(xy, X));
  *folded = hb.folded;
  if (!full) return 0;
  CUDA_TRY(cudaMemcpyAsync(rs, phi, sizeof(T) * m, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaMemcpyAsync(cs, varphi, sizeof(T) * n, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaMemcpyAsync(ya, a, sizeof(T) * m, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaMemcpyAsync(yb, b, sizeof(T) * n, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaMemcpyAsync(r, rb[hb.iter & 1], sizeof(T) * m, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaMemcpyAsync(s, sb[hb.iter & 1], sizeof(T) * n, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  *alpha = hb.alpha;
  *beta = hb.beta;
  *iter = hb.iter;
  return 0;
}


// ---- engine pass (FusedEngine<T>, fused.hpp:127-165) -------------------
template <class T>
int Session<T>::engine_pass(T* xy, const T* cost, const T* rs, const T* cs, T rho_, int mode, bool dual, bool dx, bool deterministic, T* row_sums, T* col_sums, drotb_pass_out* out) {
  RC_TRY(upload_matrix(X, xy, false));
  RC_TRY(upload_matrix(C, cost, false));
  CUDA_TRY(cudaMemcpyAsync(phi, rs, sizeof(T) * m, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(varphi, cs, sizeof(T) * n, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemsetAsync(book, 0, sizeof(Book<T>), stream));
  rho = rho_;
  const bool ex = deterministic;
  if (ex && !tiles) RC_TRY(dev_alloc(&tiles, static_cast<size_t>(n_tiles)));
  PassArgs<T> pa = pass_args();
  pa.stop = nullptr;
  const bool rc = mode != kSkip;
  if (ex) launch_tile_chains<T>(pa, mode, dual && rc, dx && rc, bs, tiles, stream);
  launch_pass<T>(pa, mode, dual && rc, dx && rc, stream);
  TailArgs<T> ta = tail_args(0, mode, false, false);
  ta.want_dual = dual;
  ta.want_dx = dx;
  ta.tile_partials = tiles;
  launch_merge<T>(ta, ex, stream);
  CUDA_TRY(cudaGetLastError());
  RC_TRY(download_matrix(xy, X));
  Book<T> hb;
  RC_TRY(read_book(&hb));
  if (row_sums) CUDA_TRY(cudaMemcpy(row_sums, u, sizeof(T) * m, cudaMemcpyDeviceToHost));
  if (col_sums) CUDA_TRY(cudaMemcpy(col_sums, v, sizeof(T) * n, cudaMemcpyDeviceToHost));
  if (out) {
    out->cost_dot = rc ? static_cast<double>(hb.pass_cost) : 0.0;
    out->prev_cost_dot = rc ? static_cast<double>(hb.pass_prev) : 0.0;
    out->dual_sq = (rc && dual) ? static_cast<double>(hb.pass_dual) : 0.0;
    out->dx_sq = (rc && dx) ? static_cast<double>(hb.pass_dx) : 0.0;
    out->max_abs = static_cast<double>(hb.pass_max_abs);
    out->nonfinite = hb.pass_bad ? 1 : 0;
    out->cost_valid = rc;
    out->prev_cost_valid = rc;
    out->dual_valid = rc && dual;
    out->dx_valid = rc && dx;
    out->pad_ = 0;
  }
  return 0;
}

// explicit instantiations (the members defined in this file)
template int Session<float>::load_state(const float* xy, int32_t folded, const float* rs, const float* cs, const float* ya, const float* yb, float alpha, const float* r, const float* s, float beta, int64_t iter);
template int Session<double>::load_state(const double* xy, int32_t folded, const double* rs, const double* cs, const double* ya, const double* yb, double alpha, const double* r, const double* s, double beta, int64_t iter);
template int Session<float>::store_state(float* xy, int32_t* folded, float* rs, float* cs, float* ya, float* yb, float* alpha, float* r, float* s, float* beta, int64_t* iter, bool full);
template int Session<double>::store_state(double* xy, int32_t* folded, double* rs, double* cs, double* ya, double* yb, double* alpha, double* r, double* s, double* beta, int64_t* iter, bool full);
template int Session<float>::engine_pass(float* xy, const float* cost, const float* rs, const float* cs, float rho_, int mode, bool dual, bool dx, bool deterministic, float* row_sums, float* col_sums, drotb_pass_out* out);
template int Session<double>::engine_pass(double* xy, const double* cost, const double* rs, const double* cs, double rho_, int mode, bool dual, bool dx, bool deterministic, double* row_sums, double* col_sums, drotb_pass_out* out);

}  // namespace drotb
