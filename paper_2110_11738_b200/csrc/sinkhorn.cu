// sinkhorn.cu -- the paper's comparison baseline on the B200: plain
// (unstabilized) Sinkhorn, drot::sinkhorn_solve<T> (reference.hpp:165-288),
// SURVEY §8(f) row 4.
//
//   K = exp(-C / eta) (T), u = v = 1
//   per iteration: u = p ./ (K v), v = q ./ (K^T u)      (reference.hpp:251-260)
//   every check_every iterations (and at max_iters): err = |u.(Kv) - p|_2 +
//   |v.(K^T u) - q|_2 in double, trace row, converged when err <= tol
//   failure (numerical_failure, no plan) on any non-positive / non-finite
//   kernel entry or scaling
//   result: plan = (u_i K_ij) v_j, mu = eta log u, nu = eta log v, report =
//   residual_report (reference.hpp:186-214)
//
// Each product is one HBM-bound streaming sweep over K (4 or 8 bytes per
// entry), so an iteration moves 2*s*m*n bytes against DROT's 2.5*s*m*n
// (skip-C average) -- the paper's observation that the per-iteration costs
// of the two methods are almost identical for large problems.
// Row sums (K v): per-lane register accumulation over a column tile, one
// strip entry per tile.  Column sums (K^T u): 8 columns per lane are reduced
// across the warp with a 9-shuffle transpose-reduction, warps combined in
// shared memory, one strip entry per 1024-row block.  Fixed reduction
// orders everywhere (deterministic; summation order differs from the
// reference's sequential loops, and expf differs from libm's by <= 2 ulp:
// tolerance parity).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "drotb_host.hpp"
#include "drotb_internal.hpp"
#include "sweep.cuh"

namespace drotb {

// device time of the last Sinkhorn iteration loop on this host thread
// (CUDA events around the batches; drotb_sinkhorn_last_loop_ms)
double& sinkhorn_loop_ms() {
  static thread_local double ms = 0.0;
  return ms;
}


namespace {

constexpr int kSkW = 8;              // warps per CTA
constexpr int kSkT = kSkW * 32;      // threads per CTA
constexpr int kSkCols = 128;         // columns per tile
constexpr int kSkGroup = 8;          // columns per warp reduction

template <class T>
struct SkState {
  int64_t m, n, ld;
  int64_t n_rb, n_ct;                // row blocks (kSkT * R rows), column tiles
  T* K;
  T* u;
  T* v;
  T* rstrip;                         // [n_ct][ld]   row partials of K v
  T* cstrip;                         // [n_rb][n]    column partials of K^T u
  const T* p;
  const T* q;
  double* dscr;                      // check partials
  int32_t* flags;                    // [0] stop, [1] failed, [2] converged, [3] kernel bad
  int64_t* fail_iter;
  double* errs;                      // per check: err
};

__device__ __forceinline__ bool pos_finite(double d) {
  return d > 0 && d <= DBL_MAX;
}

// K = exp(-C / eta); flags[3] = 1 if any entry is not positive and finite
template <class T>
__global__ void sk_kernel_build(const T* C, T* K, int64_t m, int64_t n, int64_t ld, T eta,
                                int32_t* flags) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= ld) return;
  bool bad = false;
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
    T kv = T(0);
    if (i < m) {
      kv = exp(-C[j * ld + i] / eta);
      bad |= !pos_finite(static_cast<double>(kv));
    }
    K[j * ld + i] = kv;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags + 3, 1);
}

// 9-shuffle reduction of 8 per-lane column partials across the warp: on
// return, v[0] of lanes 4c .. 4c+3 holds the warp total of column c.
template <class T>
__device__ __forceinline__ void warp_reduce8(T (&v)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const T mine = b4 ? v[k + 4] : v[k];
    const T other = b4 ? v[k] : v[k + 4];
    v[k] = mine + __shfl_xor_sync(0xffffffffu, other, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const T mine = b3 ? v[k + 2] : v[k];
    const T other = b3 ? v[k] : v[k + 2];
    v[k] = mine + __shfl_xor_sync(0xffffffffu, other, 8);
  }
  {
    const T mine = b2 ? v[1] : v[0];
    const T other = b2 ? v[0] : v[1];
    v[0] = mine + __shfl_xor_sync(0xffffffffu, other, 4);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// One sweep over K: ROWS -> z = K v (strips), COLS -> w = K^T u (strips).
template <class T, bool ROWS, bool COLS>
__global__ void __launch_bounds__(kSkT) sk_sweep(const SkState<T> s) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  if (*reinterpret_cast<volatile int*>(s.flags)) return;
  __shared__ T wpart[kSkW][kSkCols];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kSkT + threadIdx.x) * R;
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * kSkCols;
  const int64_t c1 = imin64(s.n, c0 + kSkCols);
  const bool live = row0 < s.m;  // ld is a multiple of 32: whole vectors, pad rows are 0
  T uu[R], racc[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    uu[t] = (COLS && live) ? s.u[row0 + t] : T(0);  // u pad entries are 0
    racc[t] = T(0);
  }
  for (int64_t j0 = c0; j0 < c1; j0 += kSkGroup) {
    V kv[kSkGroup];
#pragma unroll
    for (int g = 0; g < kSkGroup; ++g)
      kv[g] = (live && j0 + g < c1) ? __ldcs(reinterpret_cast<const V*>(s.K + (j0 + g) * s.ld + row0))
                                    : vzero<T>();
    T cp[kSkGroup];
#pragma unroll
    for (int g = 0; g < kSkGroup; ++g) {
      T k[R];
      unpack(kv[g], k);
      if (ROWS) {
        const T vj = j0 + g < c1 ? __ldg(s.v + j0 + g) : T(0);
#pragma unroll
        for (int t = 0; t < R; ++t) racc[t] += k[t] * vj;
      }
      if (COLS) {
        T acc = T(0);
#pragma unroll
        for (int t = 0; t < R; ++t) acc += k[t] * uu[t];
        cp[g] = acc;
      }
    }
    if (COLS) {
      warp_reduce8(cp, lane);
      if ((lane & 3) == 0) wpart[warp][j0 - c0 + (lane >> 2)] = cp[0];
    }
  }
  if (ROWS && live)
    *reinterpret_cast<V*>(s.rstrip + blockIdx.y * s.ld + row0) = pack4(racc);
  if (COLS) {
    __syncthreads();
    for (int c = threadIdx.x; c < c1 - c0; c += kSkT) {
      T tot = T(0);
#pragma unroll
      for (int w = 0; w < kSkW; ++w) tot += wpart[w][c];
      s.cstrip[blockIdx.x * s.n + c0 + c] = tot;
    }
  }
}

// u = p ./ (K v) (rows) or v = q ./ (K^T u) (columns) from the strips;
// a non-positive / non-finite scaling stops the run (reference.hpp:254-260)
template <class T, bool ROWS>
__global__ void sk_update(const SkState<T> s, int64_t iter) {
  if (*reinterpret_cast<volatile int*>(s.flags)) return;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t len = ROWS ? s.m : s.n;
  bool bad = false;
  if (idx < len) {
    T acc = T(0);
    if (ROWS)
      for (int64_t g = 0; g < s.n_ct; ++g) acc += s.rstrip[g * s.ld + idx];
    else
      for (int64_t g = 0; g < s.n_rb; ++g) acc += s.cstrip[g * s.n + idx];
    const T val = (ROWS ? s.p[idx] : s.q[idx]) / acc;
    if (ROWS)
      s.u[idx] = val;
    else
      s.v[idx] = val;
    bad = !pos_finite(static_cast<double>(val));
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) {
    atomicOr(s.flags + 1, 1);
    atomicOr(s.flags, 1);  // stop: later kernels of the batch return at once
    atomicMin(reinterpret_cast<unsigned long long*>(s.fail_iter),
              static_cast<unsigned long long>(iter + 1));
  }
}

// The check of reference.hpp:262-283 from a BOTH sweep: row_err and col_err
// partials in double, then (last block) err, its trace slot and the stop.
template <class T>
__global__ void sk_check(const SkState<T> s, int64_t iter, int64_t slot, double tol,
                         unsigned* ticket) {
  if (*reinterpret_cast<volatile int*>(s.flags)) return;
  __shared__ double sh[2][32];
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double re = 0, ce = 0;
  if (idx < s.m) {
    T acc = T(0);
    for (int64_t g = 0; g < s.n_ct; ++g) acc += s.rstrip[g * s.ld + idx];
    const double d = static_cast<double>(s.u[idx] * acc) - static_cast<double>(s.p[idx]);
    re = d * d;
  } else if (idx < s.m + s.n) {
    const int64_t j = idx - s.m;
    T acc = T(0);
    for (int64_t g = 0; g < s.n_rb; ++g) acc += s.cstrip[g * s.n + j];
    const double d = static_cast<double>(s.v[j] * acc) - static_cast<double>(s.q[j]);
    ce = d * d;
  }
  re = warp_sum(re);
  ce = warp_sum(ce);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][warp] = re;
    sh[1][warp] = ce;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      a += sh[0][w];
      b += sh[1][w];
    }
    s.dscr[2 * blockIdx.x] = a;
    s.dscr[2 * blockIdx.x + 1] = b;
  }
  if (!last_block(ticket)) return;
  if (threadIdx.x != 0) return;
  *ticket = 0u;
  double a = 0, b = 0;
  for (unsigned k = 0; k < gridDim.x; ++k) {
    a += s.dscr[2 * k];
    b += s.dscr[2 * k + 1];
  }
  const double err = sqrt(a) + sqrt(b);
  s.errs[slot] = err;
  if (!(err <= DBL_MAX)) {  // non-finite error: numerical failure
    s.flags[1] = 1;
    *s.fail_iter = iter + 1;
  } else if (err <= tol) {
    s.flags[2] = 1;
    *s.fail_iter = iter + 1;  // iteration count at convergence
  }
  if (s.flags[1] || s.flags[2]) s.flags[0] = 1;
}

// plan = (u_i K_ij) v_j in place of K
template <class T>
__global__ void sk_plan(T* K, const T* u, const T* v, int64_t m, int64_t n, int64_t ld) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const T ui = u[i];
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) K[j * ld + i] = (ui * K[j * ld + i]) * v[j];
}

}  // namespace

template <class T>
int sinkhorn_t(const T* C, int64_t m, int64_t n, const T* p, const T* q, T eta, double tol,
               int64_t max_iters, int64_t check_every, int32_t exact_report, T* plan, T* mu,
               T* nu, drotb_report* rep, drotb_trace_row* trace, int64_t trace_cap,
               int64_t* trace_len, int64_t* iterations, int32_t* status, double* wall) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  if (m <= 0 || n <= 0) return set_error(DROTB_ERRC_EMPTY_DIMENSION, "sinkhorn: empty dimension");
  if (!(eta > T(0))) return set_error(DROTB_ERRC_BAD_CONFIG, "sinkhorn eta must be positive");
  for (int64_t i = 0; i < m; ++i)
    if (!(p[i] > T(0))) return set_error(DROTB_ERRC_ZERO_MARGINAL, "sinkhorn requires p > 0");
  for (int64_t j = 0; j < n; ++j)
    if (!(q[j] > T(0))) return set_error(DROTB_ERRC_ZERO_MARGINAL, "sinkhorn requires q > 0");
  if (check_every < 1) check_every = 1;
  constexpr int R = 16 / sizeof(T);
  SkState<T> s;
  std::memset(&s, 0, sizeof(s));
  s.m = m;
  s.n = n;
  s.ld = round_up(m, 32);
  s.n_rb = (m + int64_t(kSkT) * R - 1) / (int64_t(kSkT) * R);
  s.n_ct = (n + kSkCols - 1) / kSkCols;
  const size_t mat = static_cast<size_t>(s.ld) * static_cast<size_t>(n);
  const int64_t n_checks = std::max<int64_t>(max_iters, 0) / check_every + 2;
  const int64_t check_blocks = (m + n + 255) / 256;
  // one allocation: C/K, vectors, strips, scratch
  size_t bytes = 0;
  auto take = [&](size_t b) { size_t off = bytes; bytes += (b + 255) / 256 * 256; return off; };
  const size_t oK = take(sizeof(T) * mat), oU = take(sizeof(T) * s.ld), oV = take(sizeof(T) * n),
               oP = take(sizeof(T) * s.ld), oQ = take(sizeof(T) * n),
               oR = take(sizeof(T) * s.n_ct * s.ld), oC = take(sizeof(T) * s.n_rb * n),
               oD = take(sizeof(double) * 2 * check_blocks),
               oF = take(sizeof(int32_t) * 4 + 16), oI = take(sizeof(int64_t)),
               oE = take(sizeof(double) * n_checks), oT = take(sizeof(unsigned));
  char* base = nullptr;
  cudaStream_t st = nullptr;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&base), bytes));
  std::unique_ptr<char, decltype(&cudaFree)> hold(base, &cudaFree);
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> hs(st, &cudaStreamDestroy);
  s.K = reinterpret_cast<T*>(base + oK);
  s.u = reinterpret_cast<T*>(base + oU);
  s.v = reinterpret_cast<T*>(base + oV);
  T* dp = reinterpret_cast<T*>(base + oP);
  T* dq = reinterpret_cast<T*>(base + oQ);
  s.p = dp;
  s.q = dq;
  s.rstrip = reinterpret_cast<T*>(base + oR);
  s.cstrip = reinterpret_cast<T*>(base + oC);
  s.dscr = reinterpret_cast<double*>(base + oD);
  s.flags = reinterpret_cast<int32_t*>(base + oF);
  s.fail_iter = reinterpret_cast<int64_t*>(base + oI);
  s.errs = reinterpret_cast<double*>(base + oE);
  unsigned* ticket = reinterpret_cast<unsigned*>(base + oT);
  CUDA_TRY(cudaMemsetAsync(base, 0, bytes, st));  // pad rows / entries are zero
  // C -> the K buffer (ld-pitched), then K = exp(-C/eta) in place
  CUDA_TRY(cudaMemcpy2DAsync(s.K, sizeof(T) * s.ld, C, sizeof(T) * m, sizeof(T) * m, n,
                             cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dp, p, sizeof(T) * m, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dq, q, sizeof(T) * n, cudaMemcpyHostToDevice, st));
  const int64_t big = std::numeric_limits<int64_t>::max();
  CUDA_TRY(cudaMemcpyAsync(s.fail_iter, &big, sizeof(big), cudaMemcpyHostToDevice, st));
  {
    dim3 g(static_cast<unsigned>((s.ld + 255) / 256), static_cast<unsigned>(std::min<int64_t>(n, 1024)));
    sk_kernel_build<T><<<g, 256, 0, st>>>(s.K, s.K, m, n, s.ld, eta, s.flags);
  }
  {
    std::vector<T> ones(static_cast<size_t>(std::max(m, n)), T(1));
    CUDA_TRY(cudaMemcpyAsync(s.u, ones.data(), sizeof(T) * m, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(s.v, ones.data(), sizeof(T) * n, cudaMemcpyHostToDevice, st));
    int32_t f[4];
    CUDA_TRY(cudaMemcpyAsync(f, s.flags, sizeof(f), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (f[3]) {  // bad kernel: numerical_failure at iteration 0, no plan
      if (status) *status = DROTB_NUMERICAL_FAILURE;
      if (iterations) *iterations = 0;
      if (trace_len) *trace_len = 0;
      const double nan = std::numeric_limits<double>::quiet_NaN();
      if (rep) *rep = drotb_report{nan, -1.0, -1.0, nan};
      if (plan) std::memset(plan, 0, sizeof(T) * m * n);
      if (mu) std::memset(mu, 0, sizeof(T) * m);
      if (nu) std::memset(nu, 0, sizeof(T) * n);
      if (wall) *wall = std::chrono::duration<double>(clk::now() - t0).count();
      count_launch(1);
      return 0;
    }
  }
  const dim3 sg(static_cast<unsigned>(s.n_rb), static_cast<unsigned>(s.n_ct));
  const unsigned ub = static_cast<unsigned>((m + 255) / 256), vb = static_cast<unsigned>((n + 255) / 256);
  int64_t launches = 1;
  int64_t checks = 0;
  int32_t hflags[4] = {0, 0, 0, 0};
  // batches of check_every iterations; the host reads a batch's stop flags
  // one batch behind (the next batch is already queued: every kernel returns
  // at once after a stop), so the device never idles on the poll
  int32_t* hpin = nullptr;
  CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&hpin), 8 * sizeof(int32_t)));
  std::unique_ptr<int32_t, decltype(&cudaFreeHost)> hold_pin(hpin, &cudaFreeHost);
  cudaEvent_t evb[2] = {nullptr, nullptr}, lt[2] = {nullptr, nullptr};
  for (auto* e : {&evb[0], &evb[1]}) CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (auto* e : {&lt[0], &lt[1]}) CUDA_TRY(cudaEventCreate(e));
  struct EvHold {
    cudaEvent_t* e;
    int k;
    ~EvHold() {
      for (int i = 0; i < k; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } hold_evb{evb, 2}, hold_lt{lt, 2};
  CUDA_TRY(cudaEventRecord(lt[0], st));
  int64_t k = 0, batch = 0;
  for (; k < max_iters;) {
    const int64_t kb = std::min(max_iters, (k / check_every + 1) * check_every);
    for (; k < kb; ++k) {
      sk_sweep<T, true, false><<<sg, kSkT, 0, st>>>(s);
      sk_update<T, true><<<ub, 256, 0, st>>>(s, k);
      sk_sweep<T, false, true><<<sg, kSkT, 0, st>>>(s);
      sk_update<T, false><<<vb, 256, 0, st>>>(s, k);
      launches += 4;
    }
    // check at k = kb (reference.hpp:262: (k+1) % check_every == 0 || k+1 == max_iters)
    sk_sweep<T, true, true><<<sg, kSkT, 0, st>>>(s);
    sk_check<T><<<static_cast<unsigned>(check_blocks), 256, 0, st>>>(s, k - 1, checks, tol, ticket);
    launches += 2;
    ++checks;
    const int slot = static_cast<int>(batch & 1);
    CUDA_TRY(cudaMemcpyAsync(hpin + 4 * slot, s.flags, 4 * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(evb[slot], st));
    if (batch >= 1) {
      CUDA_TRY(cudaEventSynchronize(evb[slot ^ 1]));
      const int32_t* f = hpin + 4 * (slot ^ 1);
      if (f[0] || f[1]) break;
    }
    ++batch;
  }
  CUDA_TRY(cudaEventRecord(lt[1], st));
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(hflags, s.flags, sizeof(hflags), cudaMemcpyDeviceToHost));
  {
    float lms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&lms, lt[0], lt[1]));
    sinkhorn_loop_ms() = static_cast<double>(lms);
  }
  int64_t fail_iter = 0;
  CUDA_TRY(cudaMemcpy(&fail_iter, s.fail_iter, sizeof(fail_iter), cudaMemcpyDeviceToHost));
  const bool failed = hflags[1] != 0, converged = hflags[2] != 0;
  const int64_t iters = (failed || converged) ? fail_iter : k;
  // trace rows: one per completed check (the failing check included)
  std::vector<double> errs(static_cast<size_t>(checks));
  if (checks)
    CUDA_TRY(cudaMemcpy(errs.data(), s.errs, sizeof(double) * checks, cudaMemcpyDeviceToHost));
  int64_t rows = 0;
  {
    // a failed run records the checks before the failing iteration (a
    // non-finite err returns before its row is pushed, reference.hpp:274-276)
    // (batches queued behind a stop ran no check: rows end at the stop)
    const int64_t lim = failed || converged ? iters : big;
    for (int64_t c = 0; c < checks; ++c) {
      const int64_t it = std::min(max_iters, (c + 1) * check_every);
      if (failed ? it >= lim : it > lim) break;
      if (trace && rows < trace_cap) {
        drotb_trace_row& r = trace[rows];
        r.iter = it;
        r.r_primal = errs[c];
        r.r_dual = -1.0;  // kResidualNotApplicable (problem.hpp:64)
        // the reference leaves the other TraceRow fields at their defaults
        // (problem.hpp:77-85; reference.hpp:279-283)
        r.gap = r.objective = r.ergodic_objective = r.fixed_point_residual = 0.0;
      }
      ++rows;
    }
  }
  if (trace_len) *trace_len = rows;
  if (iterations) *iterations = iters;
  if (status) *status = failed ? DROTB_NUMERICAL_FAILURE : converged ? DROTB_CONVERGED : DROTB_MAX_ITERS;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  if (failed) {
    if (rep) *rep = drotb_report{nan, -1.0, -1.0, nan};
    if (plan) std::memset(plan, 0, sizeof(T) * m * n);
    if (mu) std::memset(mu, 0, sizeof(T) * m);
    if (nu) std::memset(nu, 0, sizeof(T) * n);
  } else {
    {
      dim3 g(static_cast<unsigned>((m + 255) / 256), static_cast<unsigned>(std::min<int64_t>(n, 1024)));
      sk_plan<T><<<g, 256, 0, st>>>(s.K, s.u, s.v, m, n, s.ld);
      ++launches;
    }
    std::vector<T> hu(static_cast<size_t>(m)), hv(static_cast<size_t>(n)), hmu(m), hnu(n);
    CUDA_TRY(cudaMemcpyAsync(hu.data(), s.u, sizeof(T) * m, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(hv.data(), s.v, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
    std::vector<T> hplan;
    T* pl = plan;
    if (!pl) {
      hplan.resize(static_cast<size_t>(m) * n);
      pl = hplan.data();
    }
    CUDA_TRY(cudaMemcpy2DAsync(pl, sizeof(T) * m, s.K, sizeof(T) * s.ld, sizeof(T) * m, n,
                               cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    bool duals_ok = true;
    for (int64_t i = 0; i < m; ++i) {  // mu = eta log u (reference.hpp:199-203)
      hmu[i] = eta * std::log(hu[i]);
      duals_ok = duals_ok && std::isfinite(static_cast<double>(hmu[i]));
    }
    for (int64_t j = 0; j < n; ++j) {
      hnu[j] = eta * std::log(hv[j]);
      duals_ok = duals_ok && std::isfinite(static_cast<double>(hnu[j]));
    }
    if (mu) std::memcpy(mu, hmu.data(), sizeof(T) * m);
    if (nu) std::memcpy(nu, hnu.data(), sizeof(T) * n);
    if (rep) {
      count_launch(launches);
      launches = 0;
      int rc;
      if (std::is_same<T, float>::value)
        rc = drotb_residual_report_f32(reinterpret_cast<const float*>(C), m, n,
                                       reinterpret_cast<const float*>(p),
                                       reinterpret_cast<const float*>(q),
                                       reinterpret_cast<const float*>(pl),
                                       reinterpret_cast<const float*>(hmu.data()),
                                       reinterpret_cast<const float*>(hnu.data()), exact_report, rep);
      else
        rc = drotb_residual_report_f64(reinterpret_cast<const double*>(C), m, n,
                                       reinterpret_cast<const double*>(p),
                                       reinterpret_cast<const double*>(q),
                                       reinterpret_cast<const double*>(pl),
                                       reinterpret_cast<const double*>(hmu.data()),
                                       reinterpret_cast<const double*>(hnu.data()), exact_report, rep);
      if (rc) return rc;
      if (!duals_ok) rep->r_dual = rep->gap = -1.0;  // no representable certificate
    }
  }
  count_launch(launches);
  if (wall) *wall = std::chrono::duration<double>(clk::now() - t0).count();
  return 0;
}

template int sinkhorn_t<float>(const float*, int64_t, int64_t, const float*, const float*, float,
                               double, int64_t, int64_t, int32_t, float*, float*, float*,
                               drotb_report*, drotb_trace_row*, int64_t, int64_t*, int64_t*,
                               int32_t*, double*);
template int sinkhorn_t<double>(const double*, int64_t, int64_t, const double*, const double*,
                                double, double, int64_t, int64_t, int32_t, double*, double*,
                                double*, drotb_report*, drotb_trace_row*, int64_t, int64_t*,
                                int64_t*, int32_t*, double*);

}  // namespace drotb

extern "C" {

int drotb_sinkhorn_f32(const float* C, int64_t m, int64_t n, const float* p, const float* q,
                       float eta, double tol, int64_t max_iters, int64_t check_every,
                       int32_t exact_report, float* plan, float* mu, float* nu,
                       drotb_report* report, drotb_trace_row* trace, int64_t trace_cap,
                       int64_t* trace_len, int64_t* iterations, int32_t* status, double* wall) {
  drotb::clear_error();
  return drotb::sinkhorn_t<float>(C, m, n, p, q, eta, tol, max_iters, check_every, exact_report,
                                  plan, mu, nu, report, trace, trace_cap, trace_len, iterations,
                                  status, wall);
}

int drotb_sinkhorn_f64(const double* C, int64_t m, int64_t n, const double* p, const double* q,
                       double eta, double tol, int64_t max_iters, int64_t check_every,
                       int32_t exact_report, double* plan, double* mu, double* nu,
                       drotb_report* report, drotb_trace_row* trace, int64_t trace_cap,
                       int64_t* trace_len, int64_t* iterations, int32_t* status, double* wall) {
  drotb::clear_error();
  return drotb::sinkhorn_t<double>(C, m, n, p, q, eta, tol, max_iters, check_every, exact_report,
                                   plan, mu, nu, report, trace, trace_cap, trace_len, iterations,
                                   status, wall);
}

double drotb_sinkhorn_last_loop_ms(void) { return drotb::sinkhorn_loop_ms(); }

}  // extern "C"
