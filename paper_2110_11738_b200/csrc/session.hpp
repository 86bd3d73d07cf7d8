// session.hpp -- the host driver of the B200 DROT solver: Session<T> owns
// the device-resident DrotState (solver.hpp:98-114) and runs the solve loop
// of drot::solve<T> (solver.hpp:372-540) as kernels per iteration, captured
// as CUDA graphs (batches of even/odd iteration pairs, which fix the pass
// modes and the r/s ping-pong buffers).  All per-iteration decisions
// (recursions, ergodic mean, gate, exact confirm, max_iters) are taken on the
// device; the host only polls a stop flag once per batch, one batch behind.
//
// Implementation files:
//   session.cu        lifecycle, problem upload / validation, init, the loop,
//                     graphs, results (plan, duals, report, trace, support)
//   session_shard.cu  row shards: NCCL or NVLink peer-memory exchange
//   session_state.cu  external state (drot_step) and the FusedEngine pass API
//   abi.cu            errors and the C ABI of include/drotb.h
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include <nccl.h>

#include "drotb_host.hpp"
#include "drotb_internal.hpp"

namespace drotb {

// NCCL is bound at run time (dlopen "libnccl.so.2") and only when a sharded
// session is created, so the library never pins a NCCL build: inside a
// PyTorch process it shares the NCCL torch already loaded (session_shard.cu).
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  std::string err;
};
NcclApi& nccl();

// Replaces the thread's last error text (abi.cu).
void set_error_text(const std::string& what);

#define NCCL_TRY(expr)                                                        \
  do {                                                                        \
    ncclResult_t r_ = (expr);                                                 \
    if (r_ != ncclSuccess)                                                    \
      return ::drotb::set_cuda_error(DROTB_ERR_NCCL + static_cast<int>(r_),   \
                                     std::string("nccl: ") + #expr + ": " +   \
                                         ::drotb::nccl().getErrorString(r_)); \
  } while (0)

template <class P>
inline int dev_alloc(P** ptr, size_t count) {
  *ptr = nullptr;
  if (count == 0) count = 1;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(ptr), count * sizeof(P)));
  return 0;
}

// Selects a session's device for the duration of a C ABI call and restores
// the caller's current device afterwards (the caller may be torch, with its
// own current device).
class DeviceGuard {
 public:
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
    if (device >= 0 && device != prev_) {
      if (cudaSetDevice(device) == cudaSuccess) switched_ = true;
    }
  }
  ~DeviceGuard() {
    if (switched_ && prev_ >= 0) cudaSetDevice(prev_);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  int prev_ = -1;
  bool switched_ = false;
};

template <class T>
struct Session {

  int64_t m = 0, n = 0, ld = 0, m_global = 0, n_global = 0, row_begin = 0;
  drotb_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;

  T *X = nullptr, *C = nullptr, *Xout = nullptr;
  T *phi = nullptr, *varphi = nullptr, *a = nullptr, *b = nullptr;
  T *rb[2] = {nullptr, nullptr}, *sb[2] = {nullptr, nullptr};
  T *p = nullptr, *q = nullptr, *u = nullptr, *v = nullptr;
  T *ustrip = nullptr, *vstrip = nullptr, *tscr = nullptr;
  PassPartial<T>* partials = nullptr;
  PassPartial<T>* tiles = nullptr;
  double *dscr = nullptr, *terms = nullptr;
  Book<T>* book = nullptr;
  TraceRowDev* trace = nullptr;
  unsigned long long* vflags = nullptr;
  int32_t* h_stop = nullptr;  // pinned, 2 slots
  char* hpin = nullptr;       // pinned staging for small host <-> device transfers
  cudaEvent_t ev[2] = {nullptr, nullptr};

  // row sharding (multi-GPU): this rank holds rows [row_begin, row_begin+m)
  // exchange: 0 = NCCL allreduces (per-launch kernels), 1 = NVLink peer
  // memory fused into the cooperative tail (tail.cu shard_tail_kernel)
  int xmode = 0;
  char* xbuf = nullptr;            // this rank's exchange buffer (see XArgs)
  int64_t xbytes = 0, xsetup_off = 0, xsetup_bytes = 0;
  char** d_xpeers = nullptr;       // device array of the peers' buffers
  std::vector<void*> xopened;      // IPC mappings to close
  XArgs xa{};
  bool x_attached = false;
  unsigned long long xsetup_gen = 0;
  int rank = 0, world = 1;
  bool sharded = false;
  ncclComm_t comm = nullptr;
  T* pack = nullptr;      // [v (n) | sum r, |r|^2, cost, prev, dual, dx, non-finite count]
  T* pmax = nullptr;      // [max|t|]
  double* dpack = nullptr;  // [row-side update sums (4) | report sums (2) | misc]
  int32_t* dint = nullptr;

  // cooperative tail kernel (fast order, one GPU; tail.cu)
  bool coop = false, coop_graphs = false, fused_gate = true, pdl_ok = false, tail_pdl = false;
  int ctail_cap = 16;  // cluster tail: max CTAs per cluster (DROTB_CTAIL; 0 = grid tail only)
  // L2 policies (sweep.cuh): bit 0 evict_first on the streamed X / C reads
  // (measured slower: off), bit 1 evict_last on the row / column strips K1
  // leaves for the tail (default: +2 % per iteration at 10k^2, r1n)
  int l2hint = -1;  // resolved in allocate(): 2 while the strips fit a third of L2
  int tgrid = 0;
  T* tcpart = nullptr;
  double* tdpart = nullptr;
  unsigned* tbar = nullptr;
  unsigned long long* tstamps = nullptr;  // DROTB_TAIL_STAMPS profiling aid
  // fixed-point row / column sums (fp32 fast order with the cooperative tail;
  // PassArgs::fx): fx_ok = available, fx = used by the current solve (off
  // for warm starts, whose row sums have no a-priori bound)
  long long *ufx = nullptr, *vfx = nullptr;
  bool fx_ok = false, fx = false;
  long long* xacc = nullptr;  // exact accumulators of the tail (2 x kXaWords)
  bool xacc_owned = true;     // false: xacc lives in the exchange buffer (row shards)
  long long* xloc = nullptr;  // row shards: this rank's sweep scalars (2 x kXaWords)
  int64_t tc_rows = 0;        // rows the sweep tiles are sized for (0: m)

  std::vector<T> hp, hq;
  std::vector<T> hp_global;  // row shards: the whole p when known (generated problems)
  T rho = T(0);
  double rho_d = 0;
  int64_t bs = 64, tc = 256, grid_cols = 0, grid_rows64 = 0, n_partials = 0;
  int64_t tile_grid_rows = 0, n_tiles = 0, tail_blocks = 0, report_blocks = 0;
  int64_t trace_cap = 0, trace_alloc = 0;
  bool exact = false, have_problem = false, initialized = false;
  bool want_dual = true, want_dx = true, gate = true;
  int64_t h_iter = 0;
  bool h_folded = false;
  bool sharded_create = false;  // create() called from create_sharded()

  ~Session() {
    DeviceGuard g(device);
    drop_graphs();
    for (auto e : tev) cudaEventDestroy(e);
    release();
  }

  void release();

  int create(int64_t m_, int64_t n_, const drotb_config& c, bool engine = false);

  int setup_coop_tail();

  // Row shard [row_begin, row_end) of an m_global x n problem on `world`
  // ranks (one process per GPU); collectives over NCCL.
  int create_sharded(int64_t m_glob, int64_t n_, const drotb_config& c, int rk, int ws,
                     const char* id128, int64_t r0, int64_t r1, int exchange = 0);

  // peers: device pointers of the peers' exchange buffers in this process
  // (ptrs, e.g. sessions of one process on one or several GPUs) or CUDA IPC
  // handles (handles, world x 64 bytes; one process per GPU)
  int attach_peers(const uint64_t* ptrs, const char* handles);

  template <class U>
  int allreduce(U* buf, size_t count, ncclRedOp_t op);

  // Collective error agreement: every rank returns the same code.
  int agree(int local_rc, const std::string& local_msg);

  // Fast order is free to pick the u-strip width: enough column tiles for
  // ~6 waves of 4 CTAs on each of the 148 SMs (wave-quantization and
  // latency), in multiples of the 16-column staging chunk, at most 256.
  int64_t fast_tile_cols() const;

  int allocate();

  int set_stream(void* s);

  // Upload a dense column-major m x n host/device array into an ld-pitched
  // device array (pad rows zeroed).
  int upload_matrix(T* dst, const T* src, bool is_device);

  int download_matrix(T* dst, const T* src);

  // first_nonfinite / first_negative flat indices of an uploaded matrix
  int scan_matrix(const T* buf, unsigned long long* nf, unsigned long long* ng);

  // check_marginal (problem.hpp:103-117), host: sequential double sum
  static int check_marginal(const std::vector<T>& vv, const char* name, double tol);
  // check_problem's simplex_tol (problem.hpp:122-124); solve uses the default
  double simplex_tol = 1e-12;

  // set_problem + check_problem (problem.hpp:122-136)
  int set_problem(const T* C_, const T* p_, const T* q_, bool is_device,
                  bool validate);

  int resolve_rho();

  static T host_norm_sq(const std::vector<T>& x) {  // vec_norm_sq
    T acc = T(0);
    for (T e : x) acc += e * e;
    return acc;
  }

  // init_state (solver.hpp:143-186) + solve-loop bookkeeping reset
  // (solver.hpp:387-404).
  int init(const T* x0, bool x0_is_device = false);

  int pass_mode(int64_t k, bool folded, int* mode, bool* folded_after) const {
    if (cfg.engine == DROTB_ENGINE_REFERENCE) {
      if (folded) return set_error(DROTB_ERRC_FOLD_STATE_MISMATCH, "reference pass on a folded array");
      *mode = (k & 1) ? kPlain1 : kPlain0;
      *folded_after = false;
    } else if (cfg.skip_cost) {
      *mode = folded ? kSkip : kFold;
      *folded_after = !folded;
    } else {
      *mode = (k & 1) ? kPlain1 : kPlain0;
      *folded_after = folded;  // a plain pass on a folded array is not reachable
    }
    return 0;
  }

  PassArgs<T> pass_args(int64_t k = -1);

  TailArgs<T> tail_args(int64_t k, int mode, bool folded_after, bool solver);

  // One solve-loop iteration: step_impl (solver.hpp:238-307) + the
  // bookkeeping and gate of solve (solver.hpp:406-521).
  int enqueue_iteration(cudaEvent_t pass_begin = nullptr,
                        cudaEvent_t pass_end = nullptr, int* mode_out = nullptr,
                        unsigned long long* cond_out = nullptr,
                        TailArgs<T>* report_args = nullptr);

  // Graph of n_iters (even) iterations from an even, unfolded state: per
  // iteration the sweep, merge and update kernels, then an IF node whose
  // body (the exact confirm report) runs only when the update kernel's gate
  // fired.  Optional timing events bracket the graph and every sweep.
  int build_graph(int64_t n_iters, bool timed, cudaGraphExec_t* exec_out,
                  int64_t* launches_out);

  int ensure_events(size_t need) {
    while (tev.size() < need) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      tev.push_back(e);
    }
    return 0;
  }

  // cached graphs: batch graphs (untimed) and timed graphs, keyed by length
  std::vector<std::pair<int64_t, cudaGraphExec_t>> graphs, tgraphs;
  std::vector<int64_t> graph_launches, tgraph_launches;

  int get_graph(int64_t len, bool timed, cudaGraphExec_t* ex, int64_t* nl);

  void drop_graphs();

  bool graph_ok(int64_t len) const {
    return (!sharded || xmode == 1) && cfg.use_graphs && (!coop || coop_graphs) && len >= 2 &&
           (len & 1) == 0 && (h_iter & 1) == 0 && !h_folded;
  }

  int enqueue(int64_t n_iters);
  // Builds (without launching) every graph enqueue(n_iters) would use from
  // the current state, so that a timed enqueue captures nothing.
  int prepare(int64_t n_iters);
  int64_t graph_builds = 0;  // graphs captured + instantiated so far

  // Eager run of exactly n_iters iterations bracketed by CUDA events on the
  // session stream, with an event pair around every fused-sweep launch:
  // the live measurement behind bench.py's value and roofline.
  std::vector<cudaEvent_t> tev;
  int run_timed(int64_t n_iters, double* total_ms, double* pass_ms,
                int64_t* n_pass, double* pass_bytes, int64_t* launches);

  int64_t batch_iters() const {
    // ~3.5 ms of work per graph: each graph boundary breaks the sweep's
    // programmatic-launch chain and the run loop adds a stop-flag copy per
    // batch; the host reads the flag one batch behind, so a stop costs at
    // most two batches of early-exit launches.  At least 8 iterations.
    if (const char* e = std::getenv("DROTB_BATCH")) {  // tuning aid
      const int64_t v = std::atoll(e);
      if (v >= 2) return v + (v & 1);
    }
    const double bytes = 2.5 * sizeof(T) * static_cast<double>(m) * n;
    const double t_iter = bytes / 6.0e12 + 10e-6;
    int64_t bi = static_cast<int64_t>(3.5e-3 / t_iter) + 1;
    bi = std::max<int64_t>(8, std::min<int64_t>(bi, 256));
    return bi + (bi & 1);
  }

  // Runs the loop until the device raises its stop flag (converged,
  // max_iters, numerical failure).  The host polls one batch behind so the
  // GPU queue never drains.
  // Sharded confirm after a gate pause (stop == 2): the exact report's sums
  // over all ranks, then the replicated decision (stop -> 1 or back to 0).

  int sharded_report(bool always);

  int run_sharded();

  int run();


  // Small transfers through pinned staging: a pageable copy blocks inside the
  // CUDA call until the stream drains, which must not happen while another
  // shard of this process needs the driver to reach the same exchange.
  static constexpr size_t kPinBytes = 4096;
  int d2h_small(void* dst, const void* src, size_t bytes) {
    CUDA_TRY(cudaMemcpyAsync(hpin, src, bytes, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    std::memcpy(dst, hpin, bytes);
    return 0;
  }
  int h2d_small(void* dst, const void* src, size_t bytes) {
    std::memcpy(hpin, src, bytes);
    CUDA_TRY(cudaMemcpyAsync(dst, hpin, bytes, cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    return 0;
  }

  int read_book(Book<T>* hb) {
    static_assert(sizeof(Book<T>) <= kPinBytes, "Book fits the pinned staging");
    return d2h_small(hb, book, sizeof(Book<T>));
  }

  // Final status and report (solver.hpp:527-538).
  int finalize_pending();

  int finish(int32_t* status, int64_t* iterations, drotb_report* rep);

  // materialize_plan + recover_duals (solver.hpp:188-217)
  int get_plan(T* plan, T* mu, T* nu);

  // Support of the current plan: xmax = max x_ij, nnz = #{x_ij > max(abs_tau,
  // rel_tau * xmax)} (over all ranks when row-sharded).
  int support(double rel_tau, double abs_tau, int64_t* nnz, double* xmax);

  int get_trace(drotb_trace_row* out, int64_t cap, int64_t* len);

  // ---- external-state single step (drot_step, solver.hpp:361-370) --------
  int load_state(const T* xy, int32_t folded, const T* rs, const T* cs,
                 const T* ya, const T* yb, T alpha, const T* r, const T* s,
                 T beta, int64_t iter);

  int store_state(T* xy, int32_t* folded, T* rs, T* cs, T* ya, T* yb, T* alpha,
                  T* r, T* s, T* beta, int64_t* iter, bool full);

  // ---- engine pass (FusedEngine<T>, fused.hpp:127-165) -------------------
  int engine_pass(T* xy, const T* cost, const T* rs, const T* cs, T rho_,
                  int mode, bool dual, bool dx, bool deterministic, T* row_sums,
                  T* col_sums, drotb_pass_out* out);
};

template <class T>
inline Session<T>* as_session(void* s) {
  return static_cast<Session<T>*>(s);
}

}  // namespace drotb
