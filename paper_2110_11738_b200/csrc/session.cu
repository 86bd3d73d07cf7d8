// session.cu -- Session<T> (session.hpp): lifecycle, problem upload and
// validation, init_state, the solve loop (K1 + tail per iteration, CUDA
// graphs), results (plan, duals, report, trace, support).
#include "session.hpp"

namespace drotb {


template <class T>
void Session<T>::release() {
  void* bufs[] = {X, C, Xout, phi, varphi, a, b, rb[0], rb[1], sb[0], sb[1],
                  p, q, u, v, ustrip, vstrip, tscr, partials, tiles, dscr,
                  terms, book, trace, vflags, pack, pmax, dpack, dint,
                  tcpart, tdpart, tbar, tstamps, ufx, vfx, xacc_owned ? xacc : nullptr,
                  xloc};
  tstamps = nullptr;
  ufx = vfx = nullptr;
  xacc = nullptr;
  xloc = nullptr;
  xacc_owned = true;
  fx_ok = fx = false;
  tcpart = nullptr;
  tdpart = nullptr;
  tbar = nullptr;
  coop = false;
  if (comm) nccl().commDestroy(comm);
  comm = nullptr;
  for (void* ptr : xopened) cudaIpcCloseMemHandle(ptr);
  xopened.clear();
  if (xbuf) cudaFree(xbuf);
  if (d_xpeers) cudaFree(d_xpeers);
  xbuf = nullptr;
  d_xpeers = nullptr;
  x_attached = false;
  pack = pmax = nullptr;
  dpack = nullptr;
  dint = nullptr;
  for (void* ptr : bufs)
    if (ptr) cudaFree(ptr);
  X = C = Xout = phi = varphi = a = b = p = q = u = v = ustrip = vstrip =
      tscr = nullptr;
  rb[0] = rb[1] = sb[0] = sb[1] = nullptr;
  partials = tiles = nullptr;
  dscr = terms = nullptr;
  book = nullptr;
  trace = nullptr;
  vflags = nullptr;
  if (h_stop) cudaFreeHost(h_stop);
  h_stop = nullptr;
  if (hpin) cudaFreeHost(hpin);
  hpin = nullptr;
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  ev[0] = ev[1] = nullptr;
  if (own_stream && stream) cudaStreamDestroy(stream);
  stream = nullptr;
  own_stream = false;
}


template <class T>
int Session<T>::create(int64_t m_, int64_t n_, const drotb_config& c, bool engine) {
  if (m_ <= 0 || n_ <= 0)
    return set_error(DROTB_ERRC_EMPTY_DIMENSION, "cost matrix has an empty dimension");
  cfg = c;
  if (const char* e = std::getenv("DROTB_NO_GRAPHS"))  // profiling aid (ncu)
    if (e[0] == '1') cfg.use_graphs = 0;
  m = m_global = m_;
  n = n_global = n_;
  DeviceGuard dg(cfg.device);  // the caller's current device is restored on return
  CUDA_TRY(cudaGetDevice(&device));
  CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  own_stream = true;
  exact = cfg.order == DROTB_ORDER_REFERENCE;
  bs = std::max<int64_t>(1, cfg.block_rows);
  tc = bs * std::max<int64_t>(1, cfg.work_size);
  if (!exact && !engine) tc = fast_tile_cols();
  RC_TRY(allocate());
  if (cfg.record_trace) {  // sized here so that init() (collective when sharded) never allocates
    const int64_t te = std::max<int64_t>(1, cfg.trace_every);
    trace_alloc = std::min<int64_t>(std::max<int64_t>(cfg.max_iters, 0) / te + 1, int64_t(1) << 23);
    RC_TRY(dev_alloc(&trace, static_cast<size_t>(trace_alloc)));
  }
  if (!exact && !engine && !sharded_create) {
    // default: K1 + the cooperative tail kernel; DROTB_TAIL=legacy selects
    // the three tail kernels (merge / update / report) of the exact order
    const char* tl = std::getenv("DROTB_TAIL");
    if (!(tl && tl[0] == 'l')) RC_TRY(setup_coop_tail());
  }
  return 0;
}


template <class T>
int Session<T>::setup_coop_tail() {
  if (const char* e = std::getenv("DROTB_TAIL_GATE")) fused_gate = e[0] != 'e';
  // K1 as a programmatic dependent of the tail: its CTAs issue their first
  // X / C ring stages while the tail finishes (DROTB_PDL=0 disables)
  pdl_ok = true;
  if (const char* e = std::getenv("DROTB_PDL")) pdl_ok = e[0] == '1';
  // the tail as a programmatic dependent of the sweep (opt-in, DROTB_TAIL_PDL=1;
  // probed below: a cooperative launch must accept the attribute).  Measured
  // slower: 180.1 vs 177.0 us per iteration at 10k^2 fp32, 24.3 vs 23.0 at
  // 1000^2 fp64 (r2 timeline) -- tail CTAs parked beside the last sweep wave
  tail_pdl = false;
  if (const char* e = std::getenv("DROTB_TAIL_PDL")) tail_pdl = e[0] == '1';
  // the tail as one thread-block cluster where m + n fits it (tail.cu KC);
  // DROTB_CTAIL=0: always the grid tail, =8: clusters of at most 8 CTAs
  ctail_cap = 16;
  if (const char* e = std::getenv("DROTB_CTAIL")) ctail_cap = std::atoi(e) >= 16 ? 16 : (std::atoi(e) >= 8 ? 8 : 0);
  tgrid = tail_grid<T>(device);
  if (tgrid <= 0) return 0;
  const size_t gp = static_cast<size_t>((tgrid + 31) / 32 * 32);  // value-major partials (tail.cu)
  RC_TRY(dev_alloc(&tcpart, gp * 16));
  RC_TRY(dev_alloc(&tdpart, gp * kTailDSlots));
  RC_TRY(dev_alloc(&tbar, 1024));  // top count, generation, 16 group counters (tail.cu)
  CUDA_TRY(cudaMemsetAsync(tbar, 0, 1024 * sizeof(unsigned), stream));
  if (const char* e = std::getenv("DROTB_TAIL_STAMPS"))
    if (e[0] == '1') {
      RC_TRY(dev_alloc(&tstamps, kStampWords));
      std::vector<unsigned long long> init(kStampWords);
      for (int k = 0; k < kStampWords; ++k) init[k] = (k & 1) ? 0ull : ~0ull;
      CUDA_TRY(cudaMemcpy(tstamps, init.data(), sizeof(unsigned long long) * kStampWords,
                          cudaMemcpyHostToDevice));
    }
  if (!sharded || xmode == 1) {
    // exact accumulators of the tail (every scalar sum; for row shards they
    // move into the peer-visible exchange buffer, create_sharded)
    RC_TRY(dev_alloc(&xacc, 2 * static_cast<size_t>(kXaWords)));
    CUDA_TRY(cudaMemsetAsync(xacc, 0, sizeof(long long) * 2 * kXaWords, stream));
    // fixed-point row / column sums (one word per sum in fp32, a hi / lo
    // pair in fp64); the shard tail merges strips.  DROTB_FX=0 disables
    const char* e = std::getenv("DROTB_FX");
    if (!(e && e[0] == '0')) {
      const size_t w = sizeof(T) == 4 ? 1 : 2;
      RC_TRY(dev_alloc(&ufx, w * static_cast<size_t>(ld)));
      RC_TRY(dev_alloc(&vfx, w * static_cast<size_t>(n)));
      CUDA_TRY(cudaMemsetAsync(ufx, 0, sizeof(long long) * w * ld, stream));
      CUDA_TRY(cudaMemsetAsync(vfx, 0, sizeof(long long) * w * n, stream));
      fx_ok = true;
    }
  }
  CUDA_TRY(cudaStreamSynchronize(stream));
  coop = true;
  // can a cooperative launch be captured into a graph here?  (probe on a
  // private stream; the captured launch is never executed)
  // (with the programmatic attribute first; without it if that fails)
  coop_graphs = false;
  cudaStream_t ps = nullptr;
  if (cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking) == cudaSuccess) {
    for (int attempt = 0; attempt < 2 && !coop_graphs; ++attempt) {
      if (attempt == 1) {
        if (!tail_pdl) break;
        tail_pdl = false;
      }
      cudaGraph_t gph = nullptr;
      if (cudaStreamBeginCapture(ps, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        TailArgs<T> ta = tail_args(0, kFold, true, true);
        const cudaError_t le = launch_tail<T>(ta, tcpart, tdpart, tbar, tgrid, ps);
        count_launch(-1);
        const cudaError_t ce = cudaStreamEndCapture(ps, &gph);
        if (le == cudaSuccess && ce == cudaSuccess && gph) {
          cudaGraphExec_t ex = nullptr;
          if (cudaGraphInstantiate(&ex, gph, 0) == cudaSuccess) {
            coop_graphs = true;
            cudaGraphExecDestroy(ex);
          }
        }
        if (gph) cudaGraphDestroy(gph);
      }
      (void)cudaGetLastError();
    }
    cudaStreamDestroy(ps);
  }
  (void)cudaGetLastError();  // a failed probe leaves no sticky error
  return 0;
}


// Fast order is free to pick the u-strip width: enough column tiles for
// ~6 waves of 4 CTAs on each of the 148 SMs (wave-quantization and
// latency), in multiples of the 16-column staging chunk, at most 256.
template <class T>
int64_t Session<T>::fast_tile_cols() const {
  if (const char* e = std::getenv("DROTB_TC")) {  // tuning aid (any even width)
    const int64_t v = std::atoll(e);
    if (v >= 2) return round_up(v, 2);
  }
  constexpr int R = 16 / sizeof(T);
  const int64_t rows_cta = int64_t(kWarpsPerCta) * 32 * R;
  // row shards: from the global row count, so that every rank (and the one
  // GPU solve) uses the same sweep tiles -- the per-CTA sums, and so the
  // trajectory, are then independent of the GPU count
  const int64_t rows = tc_rows > 0 ? tc_rows : m;
  const int64_t row_ctas = (rows + rows_cta - 1) / rows_cta;
  const int64_t target = 148 * 4 * 6;
  const int64_t col_tiles = std::max<int64_t>(1, (target + row_ctas - 1) / row_ctas);
  const int64_t w = round_up((n + col_tiles - 1) / col_tiles, kChunkCols);
  return std::min<int64_t>(256, std::max<int64_t>(kChunkCols, w));
}


template <class T>
int Session<T>::allocate() {
  ld = round_up(m, 32);
  constexpr int R = 16 / sizeof(T);
  const int64_t rows_cta = int64_t(kWarpsPerCta) * 32 * R;
  grid_cols = (n + tc - 1) / tc;
  grid_rows64 = (m + kVBlockRows - 1) / kVBlockRows;
  {
    const double strip_bytes =
        static_cast<double>(sizeof(T)) * (static_cast<double>(grid_cols) * round_up(m, 32) +
                                          static_cast<double>(grid_rows64) * n);
    const char* e = std::getenv("DROTB_L2HINT");
    l2hint = e ? std::atoi(e) : (strip_bytes <= 40e6 ? 2 : 0);
  }
  n_partials = ((m + rows_cta - 1) / rows_cta) * grid_cols;
  tile_grid_rows = (m + bs - 1) / bs;
  n_tiles = tile_grid_rows * grid_cols;
  tail_blocks = (m + n + 255) / 256;
  report_blocks = 148 * 8 + (m + 256 * R - 1) / (256 * R) + 1;  // report_fast_kernel grid bound
  const size_t mat = static_cast<size_t>(ld) * static_cast<size_t>(n);
  RC_TRY(dev_alloc(&X, mat));
  RC_TRY(dev_alloc(&C, mat));
  RC_TRY(dev_alloc(&phi, ld));
  RC_TRY(dev_alloc(&a, ld));
  RC_TRY(dev_alloc(&rb[0], ld));
  RC_TRY(dev_alloc(&rb[1], ld));
  RC_TRY(dev_alloc(&p, ld));
  RC_TRY(dev_alloc(&u, ld));
  RC_TRY(dev_alloc(&varphi, n));
  RC_TRY(dev_alloc(&b, n));
  RC_TRY(dev_alloc(&sb[0], n));
  RC_TRY(dev_alloc(&sb[1], n));
  RC_TRY(dev_alloc(&q, n));
  RC_TRY(dev_alloc(&v, n));
  RC_TRY(dev_alloc(&ustrip, static_cast<size_t>(grid_cols) * ld));
  RC_TRY(dev_alloc(&vstrip, static_cast<size_t>(grid_rows64) * n));
  RC_TRY(dev_alloc(&tscr, static_cast<size_t>(tail_blocks) * 8 * 3));  // merge: 8 lanes per index
  RC_TRY(dev_alloc(&partials, static_cast<size_t>(n_partials)));
  if (exact) {
    RC_TRY(dev_alloc(&tiles, static_cast<size_t>(n_tiles)));
    RC_TRY(dev_alloc(&terms, static_cast<size_t>(m + n) * 3));
  }
  RC_TRY(dev_alloc(&dscr, static_cast<size_t>(std::max(tail_blocks * 8, report_blocks * 2))));
  RC_TRY(dev_alloc(&book, 1));
  RC_TRY(dev_alloc(&vflags, 2));
  CUDA_TRY(cudaMemsetAsync(book, 0, sizeof(Book<T>), stream));
  CUDA_TRY(cudaMemsetAsync(phi, 0, sizeof(T) * ld, stream));
  CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(T) * ld, stream));
  CUDA_TRY(cudaMemsetAsync(u, 0, sizeof(T) * ld, stream));
  CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&h_stop), 2 * sizeof(int32_t)));
  CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&hpin), kPinBytes));
  CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  return 0;
}


template <class T>
int Session<T>::set_stream(void* s) {
  drop_graphs();
  if (own_stream && stream) {
    CUDA_TRY(cudaStreamSynchronize(stream));
    cudaStreamDestroy(stream);
  }
  if (s) {
    stream = static_cast<cudaStream_t>(s);
    own_stream = false;
  } else {
    CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    own_stream = true;
  }
  return 0;
}


// Upload a dense column-major m x n host/device array into an ld-pitched
// device array (pad rows zeroed).
template <class T>
int Session<T>::upload_matrix(T* dst, const T* src, bool is_device) {
  CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(T) * static_cast<size_t>(ld) * n, stream));
  CUDA_TRY(cudaMemcpy2DAsync(dst, sizeof(T) * ld, src, sizeof(T) * m,
                             sizeof(T) * m, n,
                             is_device ? cudaMemcpyDeviceToDevice
                                       : cudaMemcpyHostToDevice,
                             stream));
  return 0;
}


template <class T>
int Session<T>::download_matrix(T* dst, const T* src) {
  CUDA_TRY(cudaMemcpy2DAsync(dst, sizeof(T) * m, src, sizeof(T) * ld,
                             sizeof(T) * m, n, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  return 0;
}


// first_nonfinite / first_negative flat indices of an uploaded matrix
template <class T>
int Session<T>::scan_matrix(const T* buf, unsigned long long* nf, unsigned long long* ng) {
  const unsigned long long init[2] = {~0ull, ~0ull};
  CUDA_TRY(cudaMemcpyAsync(vflags, init, sizeof(init), cudaMemcpyHostToDevice, stream));
  launch_validate<T>(buf, m, n, ld, vflags, vflags + 1, stream);
  CUDA_TRY(cudaGetLastError());
  unsigned long long res[2];
  CUDA_TRY(cudaMemcpyAsync(res, vflags, sizeof(res), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  *nf = res[0];
  *ng = res[1];
  return 0;
}


// check_marginal (problem.hpp:103-117), host: sequential double sum
template <class T>
int Session<T>::check_marginal(const std::vector<T>& vv, const char* name, double tol) {
  if (vv.empty()) return set_error(DROTB_ERRC_EMPTY_DIMENSION, std::string(name) + " is empty");
  double sum = 0;
  for (T e : vv) {
    if (!std::isfinite(static_cast<double>(e)))
      return set_error(DROTB_ERRC_NON_FINITE_ENTRY, std::string(name) + " has a non-finite entry");
    if (e < T(0))
      return set_error(DROTB_ERRC_MARGINAL_NOT_SIMPLEX, std::string(name) + " has a negative entry");
    sum += static_cast<double>(e);
  }
  if (std::abs(sum - 1.0) > tol)
    return set_error(DROTB_ERRC_MARGINAL_NOT_SIMPLEX,
                     std::string(name) + " sums to " + std::to_string(sum));
  return 0;
}


// set_problem + check_problem (problem.hpp:122-136)
template <class T>
int Session<T>::set_problem(const T* C_, const T* p_, const T* q_, bool is_device, bool validate) {
  if (C_) RC_TRY(upload_matrix(C, C_, is_device));  // nullptr: C generated in place
  hp.assign(static_cast<size_t>(m), T(0));
  hq.assign(static_cast<size_t>(n), T(0));
  const cudaMemcpyKind k = is_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
  CUDA_TRY(cudaMemcpyAsync(hp.data(), p_, sizeof(T) * m, k, stream));
  CUDA_TRY(cudaMemcpyAsync(hq.data(), q_, sizeof(T) * n, k, stream));
  CUDA_TRY(cudaMemcpyAsync(p, hp.data(), sizeof(T) * m, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(q, hq.data(), sizeof(T) * n, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  have_problem = true;
  initialized = false;
  if (!validate) return 0;
  if (!sharded) {
    unsigned long long nf, ng;
    RC_TRY(scan_matrix(C, &nf, &ng));
    if (nf != ~0ull || ng != ~0ull) {
      if (nf < ng)
        return set_error(DROTB_ERRC_NON_FINITE_ENTRY, "cost matrix has a non-finite entry");
      return set_error(DROTB_ERRC_NEGATIVE_COST, "cost matrix has a negative entry");
    }
    RC_TRY(check_marginal(hp, "p", simplex_tol));
    RC_TRY(check_marginal(hq, "q", simplex_tol));
    return 0;
  }
  // sharded: local scans, then a collective verdict (every rank agrees);
  // the p sum is the allreduce of the rank-local sequential double sums
  int rc = 0;
  unsigned long long nf, ng;
  RC_TRY(scan_matrix(C, &nf, &ng));
  if (nf != ~0ull || ng != ~0ull)
    rc = nf < ng ? set_error(DROTB_ERRC_NON_FINITE_ENTRY, "cost matrix has a non-finite entry")
                 : set_error(DROTB_ERRC_NEGATIVE_COST, "cost matrix has a negative entry");
  double psum = 0;
  for (T e : hp) {
    if (rc) break;
    if (!std::isfinite(static_cast<double>(e)))
      rc = set_error(DROTB_ERRC_NON_FINITE_ENTRY, "p has a non-finite entry");
    else if (e < T(0))
      rc = set_error(DROTB_ERRC_MARGINAL_NOT_SIMPLEX, "p has a negative entry");
    psum += static_cast<double>(e);
  }
  const std::string msg = last_error_cstr();
  RC_TRY(agree(rc, msg));
  RC_TRY(h2d_small(dpack + 8, &psum, sizeof(double)));
  RC_TRY(allreduce(dpack + 8, 1, ncclSum));
  RC_TRY(d2h_small(&psum, dpack + 8, sizeof(double)));
  if (std::abs(psum - 1.0) > simplex_tol)
    return set_error(DROTB_ERRC_MARGINAL_NOT_SIMPLEX, "p sums to " + std::to_string(psum));
  return check_marginal(hq, "q", simplex_tol);
}


template <class T>
int Session<T>::resolve_rho() {  // DrotConfig::resolved_rho, solver.hpp:77-83
  const double r = cfg.has_rho_override
                       ? cfg.rho_override
                       : cfg.rho0 / static_cast<double>(m_global + n_global);
  if (!(r > 0) || !std::isfinite(r))
    return set_error(DROTB_ERRC_NON_POSITIVE_RHO, "resolved rho must be positive");
  rho_d = r;
  rho = static_cast<T>(r);
  return 0;
}


// init_state (solver.hpp:143-186) + solve-loop bookkeeping reset
// (solver.hpp:387-404).
template <class T>
int Session<T>::init(const T* x0, bool x0_is_device) {
  if (!have_problem) return set_error(DROTB_ERRC_BAD_CONFIG, "no problem set");
  RC_TRY(resolve_rho());
  if (xmode == 1) {  // iteration generations restart at 1 (before any collective)
    if (!x_attached) return set_error(DROTB_ERRC_BAD_CONFIG, "peers not attached");
    CUDA_TRY(cudaMemsetAsync(xbuf, 0, kXSetupFlagOff, stream));
  }
  if (tbar) CUDA_TRY(cudaMemsetAsync(tbar, 0, 1024 * sizeof(unsigned), stream));  // tail counters
  if (xacc) CUDA_TRY(cudaMemsetAsync(xacc, 0, sizeof(long long) * 2 * kXaWords, stream));
  if (xloc) CUDA_TRY(cudaMemsetAsync(xloc, 0, sizeof(long long) * 2 * kXaWords, stream));
  if (xmode == 1 && xa.off_ctr > 0)  // cross-rank counters, sums (before any collective)
    CUDA_TRY(cudaMemsetAsync(xbuf + xa.off_ctr, 0, static_cast<size_t>(xbytes - xa.off_ctr), stream));
  if (fx_ok) {  // X0 = p q' bounds every row / column sum by 1; a warm start has no bound
    const size_t w = sizeof(T) == 4 ? 1 : 2;
    CUDA_TRY(cudaMemsetAsync(ufx, 0, sizeof(long long) * w * ld, stream));
    CUDA_TRY(cudaMemsetAsync(vfx, 0, sizeof(long long) * w * n, stream));
    // (row shards always: their tail exchanges the fixed-point column sums)
    const bool want = x0 == nullptr || (sharded && xmode == 1);
    if (want != fx) drop_graphs();
    fx = want;
  }
  if (x0) {
    RC_TRY(upload_matrix(X, x0, x0_is_device));
    unsigned long long nf, ng;
    RC_TRY(scan_matrix(X, &nf, &ng));
    int rc = 0;
    if (nf != ~0ull || ng != ~0ull)
      rc = set_error(DROTB_ERRC_INVALID_INITIAL_PLAN,
                     "initial plan must be nonnegative and finite");
    const std::string msg = last_error_cstr();
    RC_TRY(agree(rc, msg));
  } else {
    launch_init_x0<T>(X, p, q, m, n, ld, stream);
  }
  CUDA_TRY(cudaMemsetAsync(phi, 0, sizeof(T) * ld, stream));
  CUDA_TRY(cudaMemsetAsync(varphi, 0, sizeof(T) * n, stream));
  CUDA_TRY(cudaMemsetAsync(a, 0, sizeof(T) * ld, stream));
  CUDA_TRY(cudaMemsetAsync(rb[0], 0, sizeof(T) * ld, stream));
  CUDA_TRY(cudaMemsetAsync(rb[1], 0, sizeof(T) * ld, stream));

  // bookkeeping
  if (cfg.record_trace) {
    const int64_t te = std::max<int64_t>(1, cfg.trace_every);
    const int64_t cap = std::min<int64_t>(std::max<int64_t>(cfg.max_iters, 0) / te + 1,
                                          int64_t(1) << 23);
    if (!trace || cap != trace_alloc) {
      // captured graphs hold the trace pointer: drop them with the buffer
      drop_graphs();
      if (trace) cudaFree(trace);
      trace = nullptr;
      RC_TRY(dev_alloc(&trace, static_cast<size_t>(cap)));
      trace_alloc = cap;
    }
    trace_cap = cap;
  } else {
    trace_cap = 0;
  }
  Book<T> hb;
  std::memset(&hb, 0, sizeof(hb));
  hb.last_cost = std::numeric_limits<double>::quiet_NaN();
  hb.last_r_dual = std::numeric_limits<double>::infinity();
  hb.prev_pass_had_cost = 1;
  hb.dual_value = 0.0;  // phi = varphi = 0
  hb.max_iters = cfg.max_iters;
  hb.check_every = std::max<int64_t>(1, cfg.check_every);
  hb.trace_every = std::max<int64_t>(1, cfg.trace_every);
  hb.trace_cap = trace_cap;
  hb.tol_primal = cfg.tol_primal;
  hb.tol_dual = cfg.tol_dual;
  hb.tol_gap = cfg.tol_gap;
  double p_norm2 = static_cast<double>(host_norm_sq(hp));
  if (sharded) {  // global |p|^2 (allreduce of the rank-local T sums)
    RC_TRY(h2d_small(dpack + 9, &p_norm2, sizeof(double)));
    RC_TRY(allreduce(dpack + 9, 1, ncclSum));
    RC_TRY(d2h_small(&p_norm2, dpack + 9, sizeof(double)));
  }
  const double p_norm = std::sqrt(p_norm2);
  const double q_norm = std::sqrt(static_cast<double>(host_norm_sq(hq)));
  hb.primal_scale = cfg.relative_tolerances ? 1.0 / (1.0 + p_norm + q_norm) : 1.0;
  hb.record_trace = cfg.record_trace ? 1 : 0;
  hb.relative = cfg.relative_tolerances ? 1 : 0;
  hb.pend_row = -1;
  hb.pend_valid = 0;
  hb.pend_buf = 0;
  {
    double sp = 0, sq = 0;
    for (T e : hp) sp += static_cast<double>(e);
    for (T e : hq) sq += static_cast<double>(e);
    if (sharded) {  // global sum p (rank-local rows)
      RC_TRY(h2d_small(dpack + 11, &sp, sizeof(double)));
      RC_TRY(allreduce(dpack + 11, 1, ncclSum));
      RC_TRY(d2h_small(&sp, dpack + 11, sizeof(double)));
    }
    hb.sum_p = sp;
    hb.sum_q = sq;
  }
  if (cfg.max_iters <= 0) hb.stop = 1;
  CUDA_TRY(cudaMemcpyAsync(book, &hb, sizeof(hb), cudaMemcpyHostToDevice, stream));
  if (sharded && xmode == 1 && x0 == nullptr &&
      static_cast<int64_t>(hp_global.size()) == m_global) {
    // X0 = p q' with the whole p known: every rank forms b, sum(a) and the
    // norms over ALL rows in the one-GPU order (the rows' a are recomputed
    // in sequence), so the start -- and with the exact tail sums the whole
    // trajectory -- is bitwise the one-GPU solve's for any rank count
    T* pgd = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&pgd), sizeof(T) * 2 * m_global, stream));
    auto freer = [this](T* ptr) { cudaFreeAsync(ptr, stream); };
    std::unique_ptr<T, decltype(freer)> hold(pgd, freer);
    CUDA_TRY(cudaMemcpyAsync(pgd, hp_global.data(), sizeof(T) * m_global,
                             cudaMemcpyHostToDevice, stream));
    T* ag = pgd + m_global;
    launch_init_sums<T>(nullptr, pgd, q, ag, b, m_global, n, 0, book, stream, nullptr, true);
    CUDA_TRY(cudaMemcpyAsync(a, ag + row_begin, sizeof(T) * m, cudaMemcpyDeviceToDevice,
                             stream));
  } else if (sharded) {  // column sums and sum(a) span all ranks
    launch_init_sums<T>(X, p, q, a, b, m, n, ld, book, stream, pack, x0 == nullptr);
    RC_TRY(allreduce(b, static_cast<size_t>(n), ncclSum));
    RC_TRY(allreduce(pack, 2, ncclSum));
    launch_init_sharded_finish<T>(b, q, n, pack, m_global + n_global, book, stream);
  } else {
    launch_init_sums<T>(X, p, q, a, b, m, n, ld, book, stream, nullptr, x0 == nullptr);
  }
  CUDA_TRY(cudaMemcpyAsync(rb[0], a, sizeof(T) * ld, cudaMemcpyDeviceToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(sb[0], b, sizeof(T) * n, cudaMemcpyDeviceToDevice, stream));
  CUDA_TRY(cudaGetLastError());
  want_dual = true;
  want_dx = cfg.record_trace != 0;
  gate = true;
  h_iter = 0;
  h_folded = false;
  initialized = true;
  return 0;
}


static bool noncoop_env() {
  const char* e = std::getenv("DROTB_TAIL_NONCOOP");
  return e && e[0] == '1';
}

template <class T>
PassArgs<T> Session<T>::pass_args(int64_t k) {
  PassArgs<T> pa;
  pa.xy = X;
  pa.cost = C;
  pa.phi = phi;
  pa.varphi = varphi;
  pa.rho = rho;
  pa.m = m;
  pa.n = n;
  pa.ld = ld;
  pa.row_begin = row_begin;
  pa.tc = tc;
  pa.ustrip = ustrip;
  pa.vstrip = vstrip;
  pa.partials = partials;
  pa.stop = &book->stop;
  pa.stamps = tstamps;
  pa.iter = &book->iter;
  pa.ufx = ufx;
  pa.vfx = vfx;
  pa.fx = fx ? 1 : 0;
  pa.pad_fx = 0;
  // the cooperative tail takes the sweep's scalars as exact sums (row
  // shards: into this rank's xloc; the tail forwards them to every rank)
  pa.xacc = nullptr;
  if (k >= 0 && coop && !exact && xacc && (!sharded || xmode == 1))
    pa.xacc = (sharded && world > 1 ? xloc : xacc) + (k & 1) * kXaWords;
  // (not for shards of one process sharing a device -- the DROTB_TAIL_NONCOOP
  // test setup: sweep CTAs parked in griddepcontrol.wait could starve a peer
  // shard's sweep that a spinning tail waits for)
  pa.pdl = (coop && pdl_ok && !(sharded && noncoop_env())) ? 1 : 0;
  pa.trigger = (coop && tail_pdl && !exact && !sharded) ? 1 : 0;
  pa.l2hint = l2hint;
  pa.pad_l2 = 0;
  return pa;
}


template <class T>
TailArgs<T> Session<T>::tail_args(int64_t k, int mode, bool folded_after, bool solver) {
  TailArgs<T> t;
  std::memset(&t, 0, sizeof(t));
  t.m = m;
  t.n = n;
  t.ld = ld;
  t.m_global = m_global;
  t.n_global = n_global;
  t.folded_after = folded_after ? 1 : 0;
  t.grid_cols = grid_cols;
  t.grid_rows64 = grid_rows64;
  t.ustrip = ustrip;
  t.vstrip = vstrip;
  t.pass_partials = partials;
  t.n_pass_partials = n_partials;
  t.p = p;
  t.q = q;
  t.u = u;
  t.v = v;
  t.r_old = rb[k & 1];
  t.r_new = rb[(k + 1) & 1];
  t.s_old = sb[k & 1];
  t.s_new = sb[(k + 1) & 1];
  t.phi = phi;
  t.varphi = varphi;
  t.a = a;
  t.b = b;
  t.rho = rho;
  t.reads_cost = mode != kSkip;
  t.want_dual = want_dual;
  t.want_dx = want_dx;
  t.solver = solver ? 1 : 0;
  t.dscratch = dscr;
  t.tscratch = tscr;
  t.terms = terms;
  t.book = book;
  t.trace = trace;
  t.tile_partials = tiles;
  t.n_tiles = n_tiles;
  t.sharded = sharded ? 1 : 0;
  t.pack = pack;
  t.pmax = pmax;
  t.dpack = dpack;
  if (sharded) t.v = pack;  // the merge writes the local v partial into the pack
  t.report_x = X;
  t.report_c = C;
  t.stamps = tstamps;
  t.fused_gate = fused_gate ? 1 : 0;
  t.tpar = static_cast<int32_t>(k & 1);
  t.ufx = ufx;
  t.vfx = vfx;
  t.fx = fx ? 1 : 0;
  t.pdl = (coop && tail_pdl && !exact && !sharded) ? 1 : 0;
  t.ctail = ctail_cap;
  t.xacc = xacc;
  std::memset(&t.x, 0, sizeof(t.x));
  t.x.world = 1;
  if (sharded && xmode == 1) t.x = xa;
  t.xloc = xloc;
  t.inv_n_d = 1.0 / static_cast<double>(n_global);
  t.inv_m_d = 1.0 / static_cast<double>(m_global);
  return t;
}


// One solve-loop iteration: step_impl (solver.hpp:238-307) + the
// bookkeeping and gate of solve (solver.hpp:406-521).
template <class T>
int Session<T>::enqueue_iteration(cudaEvent_t pass_begin, cudaEvent_t pass_end, int* mode_out, unsigned long long* cond_out, TailArgs<T>* report_args) {
  const int64_t k = h_iter;
  int mode;
  bool folded_after;
  RC_TRY(pass_mode(k, h_folded, &mode, &folded_after));
  if (mode_out) *mode_out = mode;
  PassArgs<T> pa = pass_args(k);
  if (exact) launch_tile_chains<T>(pa, mode, want_dual, want_dx, bs, tiles, stream);
  // while capturing, external records become event nodes of the graph
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (pass_begin || pass_end) CUDA_TRY(cudaStreamIsCapturing(stream, &cap));
  const unsigned evf = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  if (pass_begin) CUDA_TRY(cudaEventRecordWithFlags(pass_begin, stream, evf));
  launch_pass<T>(pa, mode, want_dual, want_dx, stream);
  if (pass_end) CUDA_TRY(cudaEventRecordWithFlags(pass_end, stream, evf));
  TailArgs<T> ta = tail_args(k, mode, folded_after, true);
  if (sharded && xmode == 1) {  // K1 + the tail with the exchange over peer memory
    CUDA_TRY(launch_tail<T>(ta, tcpart, tdpart, tbar, tgrid, stream));
    h_iter = k + 1;
    h_folded = folded_after;
    return 0;
  }
  if (coop && !exact && !sharded) {  // K1 + one cooperative tail kernel (tail.cu)
    if (tstamps) {
      static const long long delay_us = [] {
        const char* e = std::getenv("DROTB_TAIL_DELAY_US");
        return e ? std::atoll(e) : 0ll;
      }();
      if (delay_us > 0) launch_spin(static_cast<unsigned long long>(delay_us) * 1000ull, stream);
    }
    cudaError_t le = launch_tail<T>(ta, tcpart, tdpart, tbar, tgrid, stream);
    if (le != cudaSuccess && ta.pdl) {  // no programmatic cooperative launch here
      (void)cudaGetLastError();
      tail_pdl = false;
      ta.pdl = 0;
      le = launch_tail<T>(ta, tcpart, tdpart, tbar, tgrid, stream);
    }
    CUDA_TRY(le);
    h_iter = k + 1;
    h_folded = folded_after;
    return 0;
  }
  launch_merge<T>(ta, exact, stream);
  if (sharded) {  // one exchange per phase; gate pauses for confirm
    RC_TRY(allreduce(pack, static_cast<size_t>(n + 7), ncclSum));
    launch_finish<T>(ta, stream);
    launch_update<T>(ta, false, stream);
    RC_TRY(allreduce(dpack, 4, ncclSum));
    launch_gate<T>(ta, stream);
    h_iter = k + 1;
    h_folded = folded_after;
    return 0;
  }
  if (cond_out) {  // graph build: the report goes into an IF node body
    ta.cond = *cond_out;
    ta.use_cond = 1;
    launch_update<T>(ta, exact, stream);
    *report_args = ta;
  } else {
    launch_update<T>(ta, exact, stream);
    if (gate) launch_report<T>(X, C, ta, exact, false, stream);
  }
  h_iter = k + 1;
  h_folded = folded_after;
  return 0;
}


// Graph of n_iters (even) iterations from an even, unfolded state: per
// iteration the sweep, merge and update kernels, then an IF node whose
// body (the exact confirm report) runs only when the update kernel's gate
// fired.  Optional timing events bracket the graph and every sweep.
template <class T>
int Session<T>::build_graph(int64_t n_iters, bool timed, cudaGraphExec_t* exec_out, int64_t* launches_out) {
  const int64_t save_iter = h_iter;
  const bool save_folded = h_folded;
  const int64_t before = kernel_launch_count();
  if (timed) RC_TRY(ensure_events(static_cast<size_t>(2 * n_iters + 2)));
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaGraphCreate(&g, 0));
  std::unique_ptr<CUgraph_st, decltype(&cudaGraphDestroy)> hold(g, &cudaGraphDestroy);
  std::vector<cudaGraphNode_t> deps;
  const cudaStreamCaptureMode cm = cudaStreamCaptureModeThreadLocal;
  int rc = 0;
  const bool ifnode = gate && !coop;  // the cooperative tails run their own report
  for (int64_t it = 0; it < n_iters && rc == 0; ++it) {
    cudaGraphConditionalHandle h = 0;
    if (ifnode) CUDA_TRY(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
    CUDA_TRY(cudaStreamBeginCaptureToGraph(stream, g, deps.empty() ? nullptr : deps.data(),
                                           nullptr, deps.size(), cm));
    if (timed && it == 0)
      CUDA_TRY(cudaEventRecordWithFlags(tev[0], stream, cudaEventRecordExternal));
    TailArgs<T> ra;
    unsigned long long hv = static_cast<unsigned long long>(h);
    rc = enqueue_iteration(timed ? tev[2 + 2 * it] : nullptr,
                           timed ? tev[3 + 2 * it] : nullptr, nullptr,
                           ifnode ? &hv : nullptr, &ra);
    if (timed && it + 1 == n_iters && !ifnode)
      CUDA_TRY(cudaEventRecordWithFlags(tev[1], stream, cudaEventRecordExternal));
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* d = nullptr;
    size_t nd = 0;
    CUDA_TRY(cudaStreamGetCaptureInfo(stream, &cs, nullptr, nullptr, &d, &nd));
    deps.assign(d, d + nd);
    cudaGraph_t tmp;
    CUDA_TRY(cudaStreamEndCapture(stream, &tmp));
    if (rc || !ifnode) continue;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CUDA_TRY(cudaGraphAddNode(&cn, g, deps.data(), deps.size(), &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CUDA_TRY(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cm));
    launch_report<T>(X, C, ra, exact, false, stream);
    CUDA_TRY(cudaStreamEndCapture(stream, &tmp));
    deps.assign(1, cn);
    if (timed && it + 1 == n_iters) {
      CUDA_TRY(cudaStreamBeginCaptureToGraph(stream, g, deps.data(), nullptr, deps.size(), cm));
      CUDA_TRY(cudaEventRecordWithFlags(tev[1], stream, cudaEventRecordExternal));
      CUDA_TRY(cudaStreamEndCapture(stream, &tmp));
    }
  }
  h_iter = save_iter;
  h_folded = save_folded;
  if (rc) return rc;
  CUDA_TRY(cudaGraphInstantiate(exec_out, g, 0));
  // upload now: a graph's first launch otherwise carries the upload of its
  // nodes to the device (measured ~100 us for a 20-iteration graph at 10k^2,
  // inside the first timed region that launches it)
  CUDA_TRY(cudaGraphUpload(*exec_out, stream));
  ++graph_builds;
  *launches_out = kernel_launch_count() - before;
  count_launch(-*launches_out);  // captured, not launched
  return 0;
}


template <class T>
int Session<T>::get_graph(int64_t len, bool timed, cudaGraphExec_t* ex, int64_t* nl) {
  auto& gs = timed ? tgraphs : graphs;
  auto& ls = timed ? tgraph_launches : graph_launches;
  for (size_t k = 0; k < gs.size(); ++k)
    if (gs[k].first == len) {
      *ex = gs[k].second;
      *nl = ls[k];
      return 0;
    }
  RC_TRY(build_graph(len, timed, ex, nl));
  gs.emplace_back(len, *ex);
  ls.push_back(*nl);
  return 0;
}


template <class T>
void Session<T>::drop_graphs() {
  for (auto& g : graphs) cudaGraphExecDestroy(g.second);
  for (auto& g : tgraphs) cudaGraphExecDestroy(g.second);
  graphs.clear();
  tgraphs.clear();
  graph_launches.clear();
  tgraph_launches.clear();
}


template <class T>
int Session<T>::enqueue(int64_t n_iters) {
  if (!initialized) return set_error(DROTB_ERRC_BAD_CONFIG, "session not initialized");
  const int64_t bi = batch_iters();
  while (n_iters > 0) {
    if (n_iters >= bi && graph_ok(bi)) {
      cudaGraphExec_t ex;
      int64_t nl;
      RC_TRY(get_graph(bi, false, &ex, &nl));
      CUDA_TRY(cudaGraphLaunch(ex, stream));
      count_launch(nl);
      h_iter += bi;
      n_iters -= bi;
    } else if (n_iters >= 2 && graph_ok(2)) {
      cudaGraphExec_t ex;
      int64_t nl;
      RC_TRY(get_graph(2, false, &ex, &nl));
      CUDA_TRY(cudaGraphLaunch(ex, stream));
      count_launch(nl);
      h_iter += 2;
      n_iters -= 2;
    } else {
      RC_TRY(enqueue_iteration());
      n_iters -= 1;
    }
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <class T>
int Session<T>::prepare(int64_t n_iters) {
  if (!initialized) return set_error(DROTB_ERRC_BAD_CONFIG, "session not initialized");
  const int64_t save_iter = h_iter;
  const bool save_folded = h_folded;
  const int64_t bi = batch_iters();
  int rc = 0;
  while (n_iters > 0 && rc == 0) {  // the decisions of enqueue(), without launches
    cudaGraphExec_t ex;
    int64_t nl;
    if (n_iters >= bi && graph_ok(bi)) {
      rc = get_graph(bi, false, &ex, &nl);
      h_iter += bi;
      n_iters -= bi;
    } else if (n_iters >= 2 && graph_ok(2)) {
      rc = get_graph(2, false, &ex, &nl);
      h_iter += 2;
      n_iters -= 2;
    } else {
      int md;
      bool fa;
      rc = pass_mode(h_iter, h_folded, &md, &fa);
      h_folded = fa;
      h_iter += 1;
      n_iters -= 1;
    }
  }
  h_iter = save_iter;
  h_folded = save_folded;
  return rc;
}

template <class T>
int Session<T>::run_timed(int64_t n_iters, double* total_ms, double* pass_ms, int64_t* n_pass, double* pass_bytes, int64_t* launches) {
  if (!initialized) return set_error(DROTB_ERRC_BAD_CONFIG, "session not initialized");
  RC_TRY(ensure_events(static_cast<size_t>(2 * n_iters + 2)));
  const int64_t before = kernel_launch_count();
  std::vector<int> modes(static_cast<size_t>(n_iters));
  {  // modes of the iterations about to run (host-side symbolic state)
    int64_t k = h_iter;
    bool f = h_folded;
    for (int64_t it = 0; it < n_iters; ++it, ++k) {
      bool fa;
      RC_TRY(pass_mode(k, f, &modes[it], &fa));
      f = fa;
    }
  }
  if (graph_ok(n_iters)) {
    cudaGraphExec_t ex;
    int64_t nl;
    RC_TRY(get_graph(n_iters, true, &ex, &nl));
    CUDA_TRY(cudaGraphLaunch(ex, stream));
    count_launch(nl);
    h_iter += n_iters;
  } else {
    CUDA_TRY(cudaEventRecord(tev[0], stream));
    for (int64_t it = 0; it < n_iters; ++it)
      RC_TRY(enqueue_iteration(tev[2 + 2 * it], tev[3 + 2 * it]));
    CUDA_TRY(cudaEventRecord(tev[1], stream));
  }
  CUDA_TRY(cudaEventSynchronize(tev[1]));
  CUDA_TRY(cudaGetLastError());
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, tev[0], tev[1]));
  double psum = 0, bsum = 0;
  const double cells = static_cast<double>(m) * static_cast<double>(n);
  for (int64_t it = 0; it < n_iters; ++it) {
    float pm = 0;
    CUDA_TRY(cudaEventElapsedTime(&pm, tev[2 + 2 * it], tev[3 + 2 * it]));
    psum += pm;
    bsum += (modes[it] == kSkip ? 2.0 : 3.0) * sizeof(T) * cells;
  }
  if (total_ms) *total_ms = ms;
  if (pass_ms) *pass_ms = psum;
  if (n_pass) *n_pass = n_iters;
  if (pass_bytes) *pass_bytes = bsum;
  if (launches) *launches = kernel_launch_count() - before;
  return 0;
}


template <class T>
int Session<T>::run() {
  if (!initialized) return set_error(DROTB_ERRC_BAD_CONFIG, "session not initialized");
  if (sharded && xmode != 1) return run_sharded();  // NCCL: host-driven confirm pauses
  const int64_t bi = batch_iters();
  int slot = 0;
  bool pending = false;
  const int64_t limit = std::max<int64_t>(cfg.max_iters, 0) + 4 * bi + 4;
  int64_t launched = 0;
  while (true) {
    RC_TRY(enqueue(bi));
    launched += bi;
    CUDA_TRY(cudaMemcpyAsync(&h_stop[slot], &book->stop, sizeof(int32_t),
                             cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaEventRecord(ev[slot], stream));
    if (pending) {
      CUDA_TRY(cudaEventSynchronize(ev[slot ^ 1]));
      if (h_stop[slot ^ 1]) break;
    }
    pending = true;
    slot ^= 1;
    if (launched > limit) break;  // the device sets stop at max_iters
  }
  CUDA_TRY(cudaStreamSynchronize(stream));
  return 0;
}


// Final status and report (solver.hpp:527-538).
template <class T>
int Session<T>::finalize_pending() {  // coop tail: patch the last iteration's exact dual / trace terms
  if (!coop || !tdpart) return 0;
  if (sharded && xmode != 1) return 0;
  TailArgs<T> ta = tail_args(h_iter, kFold, h_folded, true);
  launch_tail_finalize<T>(ta, tdpart, tgrid, stream);
  CUDA_TRY(cudaGetLastError());
  return 0;
}


template <class T>
int Session<T>::finish(int32_t* status, int64_t* iterations, drotb_report* rep) {
  RC_TRY(finalize_pending());
  Book<T> hb;
  RC_TRY(read_book(&hb));
  int32_t st = DROTB_MAX_ITERS;
  if (hb.converged) st = DROTB_CONVERGED;
  if (hb.failed) st = DROTB_NUMERICAL_FAILURE;
  if (st == DROTB_MAX_ITERS) {
    if (sharded) {
      RC_TRY(sharded_report(true));
    } else {
      TailArgs<T> ta = tail_args(hb.iter, kPlain0, hb.folded != 0, true);
      launch_report<T>(X, C, ta, exact, true, stream);
      CUDA_TRY(cudaGetLastError());
    }
    RC_TRY(read_book(&hb));
  }
  if (status) *status = st;
  if (iterations) *iterations = hb.iterations;
  if (rep) {
    if (st == DROTB_NUMERICAL_FAILURE) {
      const double nan = std::numeric_limits<double>::quiet_NaN();
      rep->r_primal = rep->r_dual = rep->gap = rep->objective = nan;
    } else {
      rep->r_primal = hb.rep_r_primal;
      rep->r_dual = hb.rep_r_dual;
      rep->gap = hb.rep_gap;
      rep->objective = hb.rep_objective;
    }
  }
  return 0;
}


// materialize_plan + recover_duals (solver.hpp:188-217)
template <class T>
int Session<T>::get_plan(T* plan, T* mu, T* nu) {
  RC_TRY(finalize_pending());
  Book<T> hb;
  RC_TRY(read_book(&hb));
  if (plan) {
    if (!Xout) RC_TRY(dev_alloc(&Xout, static_cast<size_t>(ld) * n));
    launch_materialize<T>(X, C, Xout, rho, hb.folded, m, n, ld, stream);
    CUDA_TRY(cudaGetLastError());
    RC_TRY(download_matrix(plan, Xout));
  }
  if (mu || nu) {
    std::vector<T> hphi(static_cast<size_t>(m)), hvar(static_cast<size_t>(n));
    CUDA_TRY(cudaMemcpyAsync(hphi.data(), phi, sizeof(T) * m, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaMemcpyAsync(hvar.data(), varphi, sizeof(T) * n, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (mu)
      for (int64_t i = 0; i < m; ++i) mu[i] = hphi[i] / rho;
    if (nu)
      for (int64_t j = 0; j < n; ++j) nu[j] = hvar[j] / rho;
  }
  return 0;
}


// Support of the current plan: xmax = max x_ij, nnz = #{x_ij > max(abs_tau,
// rel_tau * xmax)} (over all ranks when row-sharded).
template <class T>
int Session<T>::support(double rel_tau, double abs_tau, int64_t* nnz, double* xmax) {
  Book<T> hb;
  RC_TRY(read_book(&hb));
  unsigned long long stats[2] = {0, 0};
  launch_plan_max<T>(X, C, rho, hb.folded, m, n, ld, vflags, stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(stats, vflags, sizeof(stats), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  double mx;
  std::memcpy(&mx, &stats[0], sizeof(mx));
  if (sharded) {
    RC_TRY(h2d_small(dpack + 10, &mx, sizeof(double)));
    RC_TRY(allreduce(dpack + 10, 1, ncclMax));
    RC_TRY(d2h_small(&mx, dpack + 10, sizeof(double)));
  }
  const double thr = std::max(abs_tau, rel_tau * mx);
  launch_plan_count<T>(X, C, rho, hb.folded, m, n, ld, thr, vflags, stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(stats, vflags, sizeof(stats), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  double cnt = static_cast<double>(stats[1]);
  if (sharded) {
    RC_TRY(h2d_small(dpack + 10, &cnt, sizeof(double)));
    RC_TRY(allreduce(dpack + 10, 1, ncclSum));
    RC_TRY(d2h_small(&cnt, dpack + 10, sizeof(double)));
  }
  if (nnz) *nnz = static_cast<int64_t>(cnt);
  if (xmax) *xmax = mx;
  return 0;
}


template <class T>
int Session<T>::get_trace(drotb_trace_row* out, int64_t cap, int64_t* len) {
  RC_TRY(finalize_pending());
  Book<T> hb;
  RC_TRY(read_book(&hb));
  if (len) *len = hb.trace_rows;
  if (out && cap > 0 && trace) {
    const int64_t cnt = std::min<int64_t>({cap, hb.trace_rows, trace_cap});
    static_assert(sizeof(TraceRowDev) == sizeof(drotb_trace_row), "trace row");
    if (cnt > 0) {
      CUDA_TRY(cudaMemcpyAsync(out, trace, sizeof(TraceRowDev) * cnt,
                               cudaMemcpyDeviceToHost, stream));
      CUDA_TRY(cudaStreamSynchronize(stream));
    }
  }
  return 0;
}

// explicit instantiations (the members defined in this file)
template void Session<float>::release();
template void Session<double>::release();
template int Session<float>::create(int64_t m_, int64_t n_, const drotb_config& c, bool engine);
template int Session<double>::create(int64_t m_, int64_t n_, const drotb_config& c, bool engine);
template int Session<float>::setup_coop_tail();
template int Session<double>::setup_coop_tail();
template int64_t Session<float>::fast_tile_cols()const;
template int64_t Session<double>::fast_tile_cols()const;
template int Session<float>::allocate();
template int Session<double>::allocate();
template int Session<float>::set_stream(void* s);
template int Session<double>::set_stream(void* s);
template int Session<float>::upload_matrix(float* dst, const float* src, bool is_device);
template int Session<double>::upload_matrix(double* dst, const double* src, bool is_device);
template int Session<float>::download_matrix(float* dst, const float* src);
template int Session<double>::download_matrix(double* dst, const double* src);
template int Session<float>::scan_matrix(const float* buf, unsigned long long* nf, unsigned long long* ng);
template int Session<double>::scan_matrix(const double* buf, unsigned long long* nf, unsigned long long* ng);
template int Session<float>::check_marginal(const std::vector<float>& vv, const char* name, double tol);
template int Session<double>::check_marginal(const std::vector<double>& vv, const char* name, double tol);
template int Session<float>::set_problem(const float* C_, const float* p_, const float* q_, bool is_device, bool validate);
template int Session<double>::set_problem(const double* C_, const double* p_, const double* q_, bool is_device, bool validate);
template int Session<float>::resolve_rho();
template int Session<double>::resolve_rho();
template int Session<float>::init(const float* x0, bool x0_is_device);
template int Session<double>::init(const double* x0, bool x0_is_device);
template PassArgs<float> Session<float>::pass_args(int64_t);
template PassArgs<double> Session<double>::pass_args(int64_t);
template TailArgs<float> Session<float>::tail_args(int64_t k, int mode, bool folded_after, bool solver);
template TailArgs<double> Session<double>::tail_args(int64_t k, int mode, bool folded_after, bool solver);
template int Session<float>::enqueue_iteration(cudaEvent_t pass_begin, cudaEvent_t pass_end, int* mode_out, unsigned long long* cond_out, TailArgs<float>* report_args);
template int Session<double>::enqueue_iteration(cudaEvent_t pass_begin, cudaEvent_t pass_end, int* mode_out, unsigned long long* cond_out, TailArgs<double>* report_args);
template int Session<float>::build_graph(int64_t n_iters, bool timed, cudaGraphExec_t* exec_out, int64_t* launches_out);
template int Session<double>::build_graph(int64_t n_iters, bool timed, cudaGraphExec_t* exec_out, int64_t* launches_out);
template int Session<float>::get_graph(int64_t len, bool timed, cudaGraphExec_t* ex, int64_t* nl);
template int Session<double>::get_graph(int64_t len, bool timed, cudaGraphExec_t* ex, int64_t* nl);
template void Session<float>::drop_graphs();
template void Session<double>::drop_graphs();
template int Session<float>::enqueue(int64_t n_iters);
template int Session<double>::enqueue(int64_t n_iters);
template int Session<float>::run_timed(int64_t n_iters, double* total_ms, double* pass_ms, int64_t* n_pass, double* pass_bytes, int64_t* launches);
template int Session<double>::run_timed(int64_t n_iters, double* total_ms, double* pass_ms, int64_t* n_pass, double* pass_bytes, int64_t* launches);
template int Session<float>::prepare(int64_t n_iters);
template int Session<double>::prepare(int64_t n_iters);
template int Session<float>::run();
template int Session<double>::run();
template int Session<float>::finalize_pending();
template int Session<double>::finalize_pending();
template int Session<float>::finish(int32_t* status, int64_t* iterations, drotb_report* rep);
template int Session<double>::finish(int32_t* status, int64_t* iterations, drotb_report* rep);
template int Session<float>::get_plan(float* plan, float* mu, float* nu);
template int Session<double>::get_plan(double* plan, double* mu, double* nu);
template int Session<float>::support(double rel_tau, double abs_tau, int64_t* nnz, double* xmax);
template int Session<double>::support(double rel_tau, double abs_tau, int64_t* nnz, double* xmax);
template int Session<float>::get_trace(drotb_trace_row* out, int64_t cap, int64_t* len);
template int Session<double>::get_trace(drotb_trace_row* out, int64_t cap, int64_t* len);

}  // namespace drotb
