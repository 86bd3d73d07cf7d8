// session.cu -- host driver of the B200 DROT solver and the C ABI of
// libdrotb200.so (include/drotb.h).
//
// The driver owns the device-resident DrotState (solver.hpp:98-114) and runs
// the solve loop of drot::solve<T> (solver.hpp:372-540) as a fixed sequence
// of kernels per iteration, captured as CUDA graphs (one graph = one
// even/odd iteration pair, which fixes the pass modes and the r/s
// ping-pong buffers).  All per-iteration decisions (recursions, ergodic
// mean, gate, exact confirm, max_iters) are taken on the device; the host
// only polls a stop flag once per batch of graphs, one batch behind.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "drotb_host.hpp"
#include "drotb_internal.hpp"

namespace drotb {

// NCCL is bound at run time (dlopen "libnccl.so.2") and only when a sharded
// session is created, so the library never pins a NCCL build: inside a
// PyTorch process it shares the NCCL torch already loaded.
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

static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("dlopen libnccl.so.2: ") + dlerror();
      return a;
    }
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.getErrorString =
        reinterpret_cast<decltype(a.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.getUniqueId && a.commInitRank && a.allReduce && a.commDestroy && a.getErrorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks the expected symbols";
    return a;
  }();
  return api;
}

// ---------------------------------------------------------------------------
// errors (errors.hpp:48-88)
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_err;
const char* const kErrcNames[] = {
    "negative_cost",  "marginal_not_simplex", "empty_dimension",
    "non_finite_entry", "shape_mismatch",     "non_positive_rho",
    "invalid_initial_plan", "non_finite_iterate", "zero_marginal",
    "too_large",      "degenerate_cost",      "dimension_mismatch",
    "fold_state_mismatch", "bad_magic",       "version_unsupported",
    "size_mismatch",  "ragged_csv",           "empty_image",
    "k_too_large",    "io_error",             "bad_config"};
}  // namespace

const char* errc_name(int errc) {
  if (errc < 0 || errc >= static_cast<int>(sizeof(kErrcNames) / sizeof(kErrcNames[0])))
    return "unknown";
  return kErrcNames[errc];
}
int set_error(int errc, const std::string& what) {
  g_err = std::string(errc_name(errc)) + ": " + what;
  return 1 + errc;
}
int set_cuda_error(int code, const std::string& what) {
  g_err = what;
  return code;
}
void clear_error() { g_err.clear(); }
const char* last_error_cstr() { return g_err.c_str(); }

#define NCCL_TRY(expr)                                                        \
  do {                                                                        \
    ncclResult_t r_ = (expr);                                                 \
    if (r_ != ncclSuccess)                                                    \
      return ::drotb::set_cuda_error(DROTB_ERR_NCCL + static_cast<int>(r_),   \
                                     std::string("nccl: ") + #expr + ": " +   \
                                         ::drotb::nccl().getErrorString(r_)); \
  } while (0)

template <class T>
constexpr ncclDataType_t nccl_type() {
  return sizeof(T) == 4 ? ncclFloat32 : ncclFloat64;
}

template <class P>
static int dev_alloc(P** ptr, size_t count) {
  *ptr = nullptr;
  if (count == 0) count = 1;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(ptr), count * sizeof(P)));
  return 0;
}

// ---------------------------------------------------------------------------
// Session<T>
// ---------------------------------------------------------------------------
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

  // persistent solver kernel (fast order, one GPU; persistent.cu)
  bool persist = false;
  int pgrid = 0;
  int64_t prows = 0, pn_rb = 0, pmax_seg = 0, pileave = 0;
  T *pustrip = nullptr, *pvstrip = nullptr, *pcpart = nullptr;
  double* pdpart = nullptr;
  unsigned* pbar = nullptr;
  int32_t *pseg_ptr = nullptr, *pseg_slot = nullptr;
  unsigned long long* psweep_ns = nullptr;
  double* pmud = nullptr;
  bool h_stale = false;  // h_iter / h_folded lag the device after persistent launches
  // cooperative tail kernel (fast order, one GPU; tail.cu)
  bool coop = false, coop_graphs = false, fused_gate = true, pdl_ok = false;
  // single-launch iteration (iter.cu; the default for order=fast on one GPU)
  bool fiter = false;
  T* vcta_buf = nullptr;  // [row block][n] per-CTA column sums (coop tail, one GPU)
  int64_t vcta_rows = 0;
  // L2 policies (sweep.cuh): bit 0 evict_first on the streamed X / C reads
  // (measured slower: off), bit 1 evict_last on the row / column strips K1
  // leaves for the tail (default: +2 % per iteration at 10k^2, r1n)
  int l2hint = -1;  // resolved in allocate(): 2 while the strips fit a third of L2
  T *ita = nullptr, *itb = nullptr, *iaprev = nullptr, *ibprev = nullptr;
  T *iugrp = nullptr, *ivcta = nullptr;
  IterRowRec<T>* irow = nullptr;
  IterColRec<T>* icol = nullptr;
  double *iurow = nullptr, *iucol = nullptr, *idpart = nullptr;
  unsigned* icnt = nullptr;
  int32_t irbn = 0, igcn = 0, igu = 1, ingrp = 1;
  int tgrid = 0;
  T* tcpart = nullptr;
  double* tdpart = nullptr;
  unsigned* tbar = nullptr;
  unsigned long long* tstamps = nullptr;  // DROTB_TAIL_STAMPS profiling aid
  bool no_persist = false;

  std::vector<T> hp, hq;
  T rho = T(0);
  double rho_d = 0;
  int64_t bs = 64, tc = 256, grid_cols = 0, grid_rows64 = 0, n_partials = 0;
  int64_t tile_grid_rows = 0, n_tiles = 0, tail_blocks = 0, report_blocks = 0;
  int64_t trace_cap = 0, trace_alloc = 0;
  bool exact = false, have_problem = false, initialized = false;
  bool want_dual = true, want_dx = true, gate = true;
  int64_t h_iter = 0;
  bool h_folded = false;

  ~Session() {
    drop_graphs();
    for (auto e : tev) cudaEventDestroy(e);
    release();
  }

  void release() {
    void* bufs[] = {X, C, Xout, phi, varphi, a, b, rb[0], rb[1], sb[0], sb[1],
                    p, q, u, v, ustrip, vstrip, tscr, partials, tiles, dscr,
                    terms, book, trace, vflags, pack, pmax, dpack, dint,
                    pustrip, pvstrip, pcpart, pdpart, pbar, pseg_ptr, pseg_slot, psweep_ns, pmud, tcpart, tdpart, tbar, tstamps,
                    ita, itb, iaprev, ibprev, iugrp, ivcta, irow, icol, iurow, iucol, idpart, icnt,
                    vcta_buf};
    vcta_buf = nullptr;
    vcta_rows = 0;
    ita = itb = iaprev = ibprev = iugrp = ivcta = nullptr;
    irow = nullptr;
    icol = nullptr;
    iurow = iucol = idpart = nullptr;
    icnt = nullptr;
    fiter = false;
    tstamps = nullptr;
    tcpart = nullptr;
    tdpart = nullptr;
    tbar = nullptr;
    coop = false;
    pustrip = pvstrip = pcpart = nullptr;
    pdpart = nullptr;
    pbar = nullptr;
    pseg_ptr = pseg_slot = nullptr;
    psweep_ns = nullptr;
    pmud = nullptr;
    persist = false;
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

  int create(int64_t m_, int64_t n_, const drotb_config& c, bool engine = false) {
    if (m_ <= 0 || n_ <= 0)
      return set_error(DROTB_ERRC_EMPTY_DIMENSION, "cost matrix has an empty dimension");
    cfg = c;
    if (const char* e = std::getenv("DROTB_NO_GRAPHS"))  // profiling aid (ncu)
      if (e[0] == '1') cfg.use_graphs = 0;
    m = m_global = m_;
    n = n_global = n_;
    if (cfg.device >= 0) CUDA_TRY(cudaSetDevice(cfg.device));
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
    if (!exact && !engine && !no_persist) {
      // default: K1 + the cooperative tail kernel; DROTB_PERSIST=1 selects the
      // persistent solver kernel, DROTB_TAIL=legacy the three tail kernels
      const char* e = std::getenv("DROTB_PERSIST");
      if (e && e[0] == '1') RC_TRY(setup_persistent());
      // DROTB_TAIL: unset / 'c' the cooperative tail kernel (tail.cu), 'f'
      // the single-launch iteration (iter.cu; measured slower at 10k^2, see
      // DESIGN.md), 'l' the three tail kernels
      const char* tl = std::getenv("DROTB_TAIL");
      if (!persist && tl && tl[0] == 'f') RC_TRY(setup_fused_iter());
      if (!persist && !(tl && (tl[0] == 'f' || tl[0] == 'l'))) RC_TRY(setup_coop_tail());
    }
    return 0;
  }

  int setup_fused_iter() {
    int64_t words = 0;
    iter_layout<T>(m, n, tc, &irbn, &igcn, &igu, &ingrp, &words);
    RC_TRY(dev_alloc(&ita, static_cast<size_t>(ld)));
    RC_TRY(dev_alloc(&itb, static_cast<size_t>(n)));
    RC_TRY(dev_alloc(&iaprev, static_cast<size_t>(ld)));
    RC_TRY(dev_alloc(&ibprev, static_cast<size_t>(n)));
    RC_TRY(dev_alloc(&iugrp, static_cast<size_t>(ingrp) * static_cast<size_t>(ld)));
    RC_TRY(dev_alloc(&ivcta, static_cast<size_t>(irbn) * static_cast<size_t>(n)));
    RC_TRY(dev_alloc(&irow, static_cast<size_t>(irbn)));
    RC_TRY(dev_alloc(&icol, static_cast<size_t>(igcn)));
    RC_TRY(dev_alloc(&iurow, static_cast<size_t>(irbn) * 4));
    RC_TRY(dev_alloc(&iucol, static_cast<size_t>(igcn) * 4));
    RC_TRY(dev_alloc(&idpart, static_cast<size_t>(kIterConfirmGrid) * 16));
    RC_TRY(dev_alloc(&icnt, static_cast<size_t>(words)));
    CUDA_TRY(cudaMemsetAsync(ita, 0, sizeof(T) * ld, stream));
    CUDA_TRY(cudaMemsetAsync(itb, 0, sizeof(T) * n, stream));
    CUDA_TRY(cudaMemsetAsync(icnt, 0, sizeof(unsigned) * words, stream));
    if (const char* e = std::getenv("DROTB_TAIL_STAMPS"))
      if (e[0] == '1') {
        RC_TRY(dev_alloc(&tstamps, 8));
        const unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
        CUDA_TRY(cudaMemcpy(tstamps, init, sizeof(init), cudaMemcpyHostToDevice));
      }
    CUDA_TRY(cudaStreamSynchronize(stream));
    fiter = true;
    return 0;
  }

  IterArgs<T> iter_args(int64_t k, int mode, bool folded_after) {
    IterArgs<T> g;
    std::memset(&g, 0, sizeof(g));
    g.pa = pass_args();
    g.t = tail_args(k, mode, folded_after, true);
    g.ta = ita;
    g.tb = itb;
    g.a_prev = iaprev;
    g.b_prev = ibprev;
    g.ugrp = iugrp;
    g.vcta = ivcta;
    g.rowrec = irow;
    g.colrec = icol;
    g.urow = iurow;
    g.ucol = iucol;
    g.cnt = icnt;
    g.dpart = idpart;
    g.rbuf0 = rb[0];
    g.rbuf1 = rb[1];
    g.sbuf0 = sb[0];
    g.sbuf1 = sb[1];
    g.rbn = irbn;
    g.gcn = igcn;
    g.gu = igu;
    g.ngrp = ingrp;
    g.off_col = 32;
    g.off_row = 32 + igcn;
    g.off_ug = 32 + igcn + irbn;
    return g;
  }

  int setup_coop_tail() {
    if (const char* e = std::getenv("DROTB_TAIL_GATE")) fused_gate = e[0] != 'e';
    // PDL for K1 after the tail: no gain in graphs (186 vs 186 us/iteration
    // at 10k^2) and it inflates the event-timed sweep, so opt-in
    if (const char* e = std::getenv("DROTB_PDL")) pdl_ok = e[0] == '1';
    tgrid = tail_grid<T>(device);
    if (tgrid <= 0) return 0;
    RC_TRY(dev_alloc(&tcpart, static_cast<size_t>(tgrid) * 16));
    RC_TRY(dev_alloc(&tdpart, static_cast<size_t>(tgrid) * 16));
    RC_TRY(dev_alloc(&tbar, 1024));  // top count, generation, 16 group counters (tail.cu)
    CUDA_TRY(cudaMemsetAsync(tbar, 0, 1024 * sizeof(unsigned), stream));
    if (const char* e = std::getenv("DROTB_TAIL_STAMPS"))
      if (e[0] == '1') {
        RC_TRY(dev_alloc(&tstamps, 8));
        const unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
        CUDA_TRY(cudaMemcpy(tstamps, init, sizeof(init), cudaMemcpyHostToDevice));
      }
    CUDA_TRY(cudaStreamSynchronize(stream));
    coop = true;
    if (!sharded && !no_persist) {  // K1 leaves one column-sum row per CTA for the tail
      const char* k1 = std::getenv("DROTB_K1");
      const char* vc = std::getenv("DROTB_VCTA");
      // opt-in: measured ~1 us per iteration slower at 10k^2 (the in-CTA
      // combine costs the sweep more than the shorter merge saves)
      if (!(k1 && k1[0] == 'r') && vc && vc[0] == '1') {
        constexpr int R = 16 / sizeof(T);
        vcta_rows = (m + int64_t(kWarpsPerCta) * 32 * R - 1) / (int64_t(kWarpsPerCta) * 32 * R);
        RC_TRY(dev_alloc(&vcta_buf, static_cast<size_t>(vcta_rows) * static_cast<size_t>(n)));
      }
    }
    // can a cooperative launch be captured into a graph here?  (probe on a
    // private stream; the captured launch is never executed)
    coop_graphs = false;
    cudaStream_t ps = nullptr;
    if (cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking) == cudaSuccess) {
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
      cudaStreamDestroy(ps);
    }
    (void)cudaGetLastError();  // a failed probe leaves no sticky error
    return 0;
  }

  // Static schedule of the persistent kernel: CTA b sweeps the flat range
  // [b*W/G, (b+1)*W/G) of the (row block, column) space; its segments get u
  // slots b*max_seg + s, listed per row block in column order (CSR).
  int setup_persistent() {
    pgrid = persistent_grid<T>(device);
    if (pgrid <= 0) return 0;  // cannot co-reside: stay on the per-launch path
    prows = rows_per_cta<T>();
    pn_rb = (m + prows - 1) / prows;
    const int64_t W = pn_rb * n, G = pgrid;
    std::vector<std::vector<int32_t>> per(static_cast<size_t>(pn_rb));
    pmax_seg = 1;
    // interleaved schedule (co-running CTAs stream contiguous column bands)
    // when whole row blocks fill >= 90 % of the grid, else flat slices
    const int64_t k = G / pn_rb;
    pileave = 0;
    if (k >= 1 && pn_rb * k * 10 >= G * 9) pileave = k;
    if (const char* e = std::getenv("DROTB_PSK_SCHED")) {
      if (e[0] == 'f') pileave = 0;
      if (e[0] == 'i' && k >= 1) pileave = k;
    }
    if (pileave > 0) {
      for (int64_t r = 0; r < pn_rb; ++r)
        for (int64_t cg = 0; cg < pileave; ++cg)
          per[static_cast<size_t>(r)].push_back(static_cast<int32_t>(r + cg * pn_rb));
    }
    for (int pass = 0; pass < (pileave > 0 ? 0 : 2); ++pass) {
      for (auto& v : per) v.clear();
      for (int64_t bi = 0; bi < G; ++bi) {
        int64_t f0 = bi * W / G;
        const int64_t f1 = (bi + 1) * W / G;
        int64_t seg = 0;
        while (f0 < f1) {
          const int64_t rbk = f0 / n, c0 = f0 - rbk * n;
          const int64_t c1 = std::min<int64_t>(n, c0 + (f1 - f0));
          per[static_cast<size_t>(rbk)].push_back(static_cast<int32_t>(bi * pmax_seg + seg));
          f0 += c1 - c0;
          ++seg;
        }
        if (pass == 0) pmax_seg = std::max<int64_t>(pmax_seg, seg);
      }
    }
    std::vector<int32_t> ptr(static_cast<size_t>(pn_rb + 1), 0), slots;
    for (int64_t r = 0; r < pn_rb; ++r) {
      ptr[static_cast<size_t>(r + 1)] = ptr[static_cast<size_t>(r)] +
                                        static_cast<int32_t>(per[static_cast<size_t>(r)].size());
      slots.insert(slots.end(), per[static_cast<size_t>(r)].begin(),
                   per[static_cast<size_t>(r)].end());
    }
    RC_TRY(dev_alloc(&pustrip, static_cast<size_t>(G * pmax_seg * prows)));
    RC_TRY(dev_alloc(&pvstrip, static_cast<size_t>(pn_rb * n)));
    RC_TRY(dev_alloc(&pcpart, static_cast<size_t>(G * 16)));
    RC_TRY(dev_alloc(&pdpart, static_cast<size_t>(G * 16)));
    RC_TRY(dev_alloc(&pbar, 2));
    RC_TRY(dev_alloc(&pseg_ptr, ptr.size()));
    RC_TRY(dev_alloc(&pseg_slot, slots.size()));
    RC_TRY(dev_alloc(&psweep_ns, 1));
    RC_TRY(dev_alloc(&pmud, static_cast<size_t>(ld)));
    CUDA_TRY(cudaMemsetAsync(pbar, 0, 2 * sizeof(unsigned), stream));
    CUDA_TRY(cudaMemsetAsync(psweep_ns, 0, sizeof(unsigned long long), stream));
    CUDA_TRY(cudaMemsetAsync(pustrip, 0, sizeof(T) * G * pmax_seg * prows, stream));
    CUDA_TRY(cudaMemcpyAsync(pseg_ptr, ptr.data(), sizeof(int32_t) * ptr.size(),
                             cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(pseg_slot, slots.data(), sizeof(int32_t) * slots.size(),
                             cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    persist = true;
    return 0;
  }

  PersistArgs<T> persist_args(int64_t iters) {
    PersistArgs<T> g;
    std::memset(&g, 0, sizeof(g));
    g.pa = pass_args();
    g.pa.stop = nullptr;
    g.a = a;
    g.b = b;
    g.p = p;
    g.q = q;
    g.rb0 = rb[0];
    g.rb1 = rb[1];
    g.sb0 = sb[0];
    g.sb1 = sb[1];
    g.m_global = m_global;
    g.n_global = n_global;
    g.rows_cta = prows;
    g.n_rb = pn_rb;
    g.max_seg = pmax_seg;
    g.ileave = pileave;
    g.ustrip = pustrip;
    g.seg_ptr = pseg_ptr;
    g.seg_slot = pseg_slot;
    g.vstrip = pvstrip;
    g.cpart = pcpart;
    g.dpart = pdpart;
    g.bar = pbar;
    g.book = book;
    g.trace = trace;
    g.iters = iters;
    g.engine_ref = cfg.engine == DROTB_ENGINE_REFERENCE ? 1 : 0;
    g.skip_cost = cfg.skip_cost ? 1 : 0;
    g.sweep_ns = psweep_ns;
    g.mud = pmud;
    return g;
  }

  int launch_persist(int64_t iters) {
    CUDA_TRY(launch_persistent<T>(persist_args(iters), pgrid, want_dx, stream));
    h_stale = true;
    return 0;
  }

  int resync() {  // host mirrors of the iteration counter and fold state
    if (!h_stale) return 0;
    Book<T> hb;
    RC_TRY(read_book(&hb));
    h_iter = hb.iter;
    h_folded = hb.folded != 0;
    h_stale = false;
    return 0;
  }

  // Row shard [row_begin, row_end) of an m_global x n problem on `world`
  // ranks (one process per GPU); collectives over NCCL.
  int create_sharded(int64_t m_glob, int64_t n_, const drotb_config& c, int rk, int ws,
                     const char* id128, int64_t r0, int64_t r1, int exchange = 0) {
    if (ws < 1 || rk < 0 || rk >= ws || r0 < 0 || r1 <= r0 || r1 > m_glob)
      return set_error(DROTB_ERRC_BAD_CONFIG, "invalid shard");
    if (c.order == DROTB_ORDER_REFERENCE)
      return set_error(DROTB_ERRC_BAD_CONFIG,
                       "order=reference reproduces the single-threaded CPU tree; "
                       "row sharding needs order=fast");
    if (exchange == 1 && ws > 32)
      return set_error(DROTB_ERRC_BAD_CONFIG, "peer-memory exchange supports <= 32 ranks");
    if (exchange == 0 && !nccl().ok)
      return set_error(DROTB_ERRC_BAD_CONFIG, "NCCL unavailable: " + nccl().err);
    drotb_config c2 = c;
    if (exchange == 0) c2.use_graphs = 0;  // NCCL iterations are enqueued eagerly (+ pause)
    no_persist = true;  // the persistent kernel has no collective phase
    RC_TRY(create(r1 - r0, n_, c2));
    m_global = m_glob;
    row_begin = r0;
    rank = rk;
    world = ws;
    sharded = true;
    RC_TRY(dev_alloc(&pack, static_cast<size_t>(n + 8)));
    RC_TRY(dev_alloc(&pmax, 2));
    RC_TRY(dev_alloc(&dpack, 16));
    RC_TRY(dev_alloc(&dint, 2));
    if (exchange == 1) {
      xmode = 1;
      RC_TRY(setup_coop_tail());
      if (!coop) return set_error(DROTB_ERRC_BAD_CONFIG, "cooperative tail unavailable");
      fused_gate = true;
      const int64_t vec = round_up(static_cast<int64_t>(sizeof(T)) * n, 16);
      xa.vec_bytes = vec;
      xa.slot_bytes = vec + 16 * 8;
      xa.buf_bytes = world * xa.slot_bytes;
      xa.world = world;
      xa.rank = rank;
      xsetup_bytes = round_up(std::max<int64_t>(n, 32) * 8, 16);
      xsetup_off = kXIterOff + 2 * xa.buf_bytes;
      xbytes = xsetup_off + 2 * world * xsetup_bytes;
      CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&xbuf), static_cast<size_t>(xbytes)));
      CUDA_TRY(cudaMemset(xbuf, 0, static_cast<size_t>(xbytes)));
      return 0;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    NCCL_TRY(nccl().commInitRank(&comm, world, id, rank));
    return 0;
  }

  // peers: device pointers of the peers' exchange buffers in this process
  // (ptrs, e.g. sessions of one process on one or several GPUs) or CUDA IPC
  // handles (handles, world x 64 bytes; one process per GPU)
  int attach_peers(const uint64_t* ptrs, const char* handles) {
    if (xmode != 1) return set_error(DROTB_ERRC_BAD_CONFIG, "session has no peer exchange");
    std::vector<char*> pv(static_cast<size_t>(world), nullptr);
    for (int r = 0; r < world; ++r) {
      if (r == rank) {
        pv[r] = xbuf;
      } else if (ptrs) {
        pv[r] = reinterpret_cast<char*>(ptrs[r]);
      } else {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + 64 * r, sizeof(h));
        void* ptr = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        xopened.push_back(ptr);
        pv[r] = static_cast<char*>(ptr);
      }
    }
    if (!d_xpeers) RC_TRY(dev_alloc(&d_xpeers, static_cast<size_t>(world)));
    CUDA_TRY(cudaMemcpy(d_xpeers, pv.data(), sizeof(char*) * world, cudaMemcpyHostToDevice));
    xa.peers = d_xpeers;
    x_attached = true;
    return 0;
  }

  template <class U>
  int allreduce(U* buf, size_t count, ncclRedOp_t op) {
    if (xmode == 1) {  // setup collective over the peer buffers (no NCCL)
      if (!x_attached) return set_error(DROTB_ERRC_BAD_CONFIG, "peers not attached");
      if (static_cast<int64_t>(count * sizeof(U)) > xsetup_bytes)
        return set_error(DROTB_ERRC_BAD_CONFIG, "setup collective too large");
      launch_xallreduce<U>(buf, buf, static_cast<int64_t>(count), op == ncclMax ? 1 : 0,
                           d_xpeers, world, rank, xsetup_off, xsetup_bytes, ++xsetup_gen,
                           stream);
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
    ncclDataType_t dt = std::is_same<U, double>::value  ? ncclFloat64
                        : std::is_same<U, float>::value ? ncclFloat32
                                                        : ncclInt32;
    NCCL_TRY(nccl().allReduce(buf, buf, count, dt, op, comm, stream));
    return 0;
  }

  // Collective error agreement: every rank returns the same code.
  int agree(int local_rc, const std::string& local_msg) {
    if (!sharded) return local_rc;
    int32_t v = local_rc;
    RC_TRY(h2d_small(dint, &v, sizeof(v)));
    RC_TRY(allreduce(dint, 1, ncclMax));
    RC_TRY(d2h_small(&v, dint, sizeof(v)));
    if (v == 0) return 0;
    if (v != local_rc) g_err = "rank " + std::to_string(rank) + ": another rank failed: " +
                               std::string(v < DROTB_ERR_CUDA ? errc_name(v - 1) : "device error");
    else g_err = local_msg;
    return v;
  }

  // Fast order is free to pick the u-strip width: enough column tiles for
  // ~6 waves of 4 CTAs on each of the 148 SMs (wave-quantization and
  // latency), in multiples of the 16-column staging chunk, at most 256.
  int64_t fast_tile_cols() const {
    if (const char* e = std::getenv("DROTB_TC")) {  // tuning aid
      const int64_t v = std::atoll(e);
      if (v >= kChunkCols) return round_up(v, kChunkCols);
    }
    constexpr int R = 16 / sizeof(T);
    const int64_t rows_cta = int64_t(kWarpsPerCta) * 32 * R;
    const int64_t row_ctas = (m + rows_cta - 1) / rows_cta;
    const int64_t target = 148 * 4 * 6;
    const int64_t col_tiles = std::max<int64_t>(1, (target + row_ctas - 1) / row_ctas);
    const int64_t w = round_up((n + col_tiles - 1) / col_tiles, kChunkCols);
    return std::min<int64_t>(256, std::max<int64_t>(kChunkCols, w));
  }

  int allocate() {
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

  int set_stream(void* s) {
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
  int upload_matrix(T* dst, const T* src, bool is_device) {
    CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(T) * static_cast<size_t>(ld) * n, stream));
    CUDA_TRY(cudaMemcpy2DAsync(dst, sizeof(T) * ld, src, sizeof(T) * m,
                               sizeof(T) * m, n,
                               is_device ? cudaMemcpyDeviceToDevice
                                         : cudaMemcpyHostToDevice,
                               stream));
    return 0;
  }

  int download_matrix(T* dst, const T* src) {
    CUDA_TRY(cudaMemcpy2DAsync(dst, sizeof(T) * m, src, sizeof(T) * ld,
                               sizeof(T) * m, n, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    return 0;
  }

  // first_nonfinite / first_negative flat indices of an uploaded matrix
  int scan_matrix(const T* buf, unsigned long long* nf, unsigned long long* ng) {
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
  static int check_marginal(const std::vector<T>& vv, const char* name) {
    if (vv.empty()) return set_error(DROTB_ERRC_EMPTY_DIMENSION, std::string(name) + " is empty");
    double sum = 0;
    for (T e : vv) {
      if (!std::isfinite(static_cast<double>(e)))
        return set_error(DROTB_ERRC_NON_FINITE_ENTRY, std::string(name) + " has a non-finite entry");
      if (e < T(0))
        return set_error(DROTB_ERRC_MARGINAL_NOT_SIMPLEX, std::string(name) + " has a negative entry");
      sum += static_cast<double>(e);
    }
    if (std::abs(sum - 1.0) > 1e-12)
      return set_error(DROTB_ERRC_MARGINAL_NOT_SIMPLEX,
                       std::string(name) + " sums to " + std::to_string(sum));
    return 0;
  }

  // set_problem + check_problem (problem.hpp:122-136)
  int set_problem(const T* C_, const T* p_, const T* q_, bool is_device,
                  bool validate) {
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
      RC_TRY(check_marginal(hp, "p"));
      RC_TRY(check_marginal(hq, "q"));
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
    const std::string msg = g_err;
    RC_TRY(agree(rc, msg));
    RC_TRY(h2d_small(dpack + 8, &psum, sizeof(double)));
    RC_TRY(allreduce(dpack + 8, 1, ncclSum));
    RC_TRY(d2h_small(&psum, dpack + 8, sizeof(double)));
    if (std::abs(psum - 1.0) > 1e-12)
      return set_error(DROTB_ERRC_MARGINAL_NOT_SIMPLEX, "p sums to " + std::to_string(psum));
    return check_marginal(hq, "q");
  }

  int resolve_rho() {  // DrotConfig::resolved_rho, solver.hpp:77-83
    const double r = cfg.has_rho_override
                         ? cfg.rho_override
                         : cfg.rho0 / static_cast<double>(m_global + n_global);
    if (!(r > 0) || !std::isfinite(r))
      return set_error(DROTB_ERRC_NON_POSITIVE_RHO, "resolved rho must be positive");
    rho_d = r;
    rho = static_cast<T>(r);
    return 0;
  }

  static T host_norm_sq(const std::vector<T>& x) {  // vec_norm_sq
    T acc = T(0);
    for (T e : x) acc += e * e;
    return acc;
  }

  // init_state (solver.hpp:143-186) + solve-loop bookkeeping reset
  // (solver.hpp:387-404).
  int init(const T* x0, bool x0_is_device = false) {
    if (!have_problem) return set_error(DROTB_ERRC_BAD_CONFIG, "no problem set");
    RC_TRY(resolve_rho());
    if (xmode == 1) {  // iteration generations restart at 1 (before any collective)
      if (!x_attached) return set_error(DROTB_ERRC_BAD_CONFIG, "peers not attached");
      CUDA_TRY(cudaMemsetAsync(xbuf, 0, kXSetupFlagOff, stream));
    }
    if (x0) {
      RC_TRY(upload_matrix(X, x0, x0_is_device));
      unsigned long long nf, ng;
      RC_TRY(scan_matrix(X, &nf, &ng));
      int rc = 0;
      if (nf != ~0ull || ng != ~0ull)
        rc = set_error(DROTB_ERRC_INVALID_INITIAL_PLAN,
                       "initial plan must be nonnegative and finite");
      const std::string msg = g_err;
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
    hb.phi_mat = 1;
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
    if (sharded) {  // column sums and sum(a) span all ranks
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
    h_stale = false;
    initialized = true;
    return 0;
  }

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

  PassArgs<T> pass_args() {
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
    pa.pdl = (coop && pdl_ok) ? 1 : 0;
    pa.l2hint = l2hint;
    pa.pad_l2 = 0;
    pa.vcta = (coop && !exact && !sharded) ? vcta_buf : nullptr;
    return pa;
  }

  TailArgs<T> tail_args(int64_t k, int mode, bool folded_after, bool solver) {
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
    if (coop && !exact && !sharded && vcta_buf) {  // the strips K1 wrote
      t.vstrip = vcta_buf;
      t.grid_rows64 = vcta_rows;
    }
    t.report_x = X;
    t.report_c = C;
    t.stamps = tstamps;
    t.fused_gate = fused_gate ? 1 : 0;
    return t;
  }

  // One solve-loop iteration: step_impl (solver.hpp:238-307) + the
  // bookkeeping and gate of solve (solver.hpp:406-521).
  int enqueue_iteration(cudaEvent_t pass_begin = nullptr,
                        cudaEvent_t pass_end = nullptr, int* mode_out = nullptr,
                        unsigned long long* cond_out = nullptr,
                        TailArgs<T>* report_args = nullptr) {
    const int64_t k = h_iter;
    int mode;
    bool folded_after;
    RC_TRY(pass_mode(k, h_folded, &mode, &folded_after));
    if (mode_out) *mode_out = mode;
    PassArgs<T> pa = pass_args();
    if (exact) launch_tile_chains<T>(pa, mode, want_dual, want_dx, bs, tiles, stream);
    // while capturing, external records become event nodes of the graph
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (pass_begin || pass_end) CUDA_TRY(cudaStreamIsCapturing(stream, &cap));
    const unsigned evf = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
    if (fiter) {  // one launch: sweep + merges + recursions + gate (iter.cu)
      const IterArgs<T> g = iter_args(k, mode, folded_after);
      if (pass_begin) CUDA_TRY(cudaEventRecordWithFlags(pass_begin, stream, evf));
      launch_iter<T>(g, mode, want_dual, want_dx, stream);
      if (pass_end) CUDA_TRY(cudaEventRecordWithFlags(pass_end, stream, evf));
      launch_iter_confirm<T>(g, stream);  // exits at once unless the gate fired
      h_iter = k + 1;
      h_folded = folded_after;
      return 0;
    }
    if (pass_begin) CUDA_TRY(cudaEventRecordWithFlags(pass_begin, stream, evf));
    launch_pass<T>(pa, mode, want_dual, want_dx, stream);
    if (pass_end) CUDA_TRY(cudaEventRecordWithFlags(pass_end, stream, evf));
    TailArgs<T> ta = tail_args(k, mode, folded_after, true);
    if (sharded && xmode == 1) {  // K1 + the tail with the fused peer exchange
      CUDA_TRY(launch_shard_tail<T>(ta, tcpart, tdpart, tbar, xa, tgrid, stream));
      h_iter = k + 1;
      h_folded = folded_after;
      return 0;
    }
    if (coop && !exact && !sharded) {  // K1 + one cooperative tail kernel (tail.cu)
      CUDA_TRY(launch_tail<T>(ta, tcpart, tdpart, tbar, tgrid, stream));
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
  int build_graph(int64_t n_iters, bool timed, cudaGraphExec_t* exec_out,
                  int64_t* launches_out) {
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
    const bool ifnode = gate && !coop && !fiter;  // the fused tails run their own report
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
    *launches_out = kernel_launch_count() - before;
    count_launch(-*launches_out);  // captured, not launched
    return 0;
  }

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

  int get_graph(int64_t len, bool timed, cudaGraphExec_t* ex, int64_t* nl) {
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

  void drop_graphs() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.second);
    for (auto& g : tgraphs) cudaGraphExecDestroy(g.second);
    graphs.clear();
    tgraphs.clear();
    graph_launches.clear();
    tgraph_launches.clear();
  }

  bool graph_ok(int64_t len) const {
    return (!sharded || xmode == 1) && cfg.use_graphs && (!coop || coop_graphs) && len >= 2 &&
           (len & 1) == 0 && (h_iter & 1) == 0 && !h_folded;
  }

  int enqueue(int64_t n_iters) {
    if (!initialized) return set_error(DROTB_ERRC_BAD_CONFIG, "session not initialized");
    if (persist && gate && n_iters > 0) return launch_persist(n_iters);
    RC_TRY(resync());
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

  // Eager run of exactly n_iters iterations bracketed by CUDA events on the
  // session stream, with an event pair around every fused-sweep launch:
  // the live measurement behind bench.py's value and roofline.
  std::vector<cudaEvent_t> tev;
  int run_timed(int64_t n_iters, double* total_ms, double* pass_ms,
                int64_t* n_pass, double* pass_bytes, int64_t* launches) {
    if (!initialized) return set_error(DROTB_ERRC_BAD_CONFIG, "session not initialized");
    RC_TRY(ensure_events(static_cast<size_t>(2 * n_iters + 2)));
    RC_TRY(resync());
    const int64_t before = kernel_launch_count();
    if (persist && gate) {
      // one persistent launch of n_iters iterations between two events; the
      // sweep phases are timed inside the kernel (%globaltimer, CTA 0)
      unsigned long long ns0 = 0, ns1 = 0;
      CUDA_TRY(cudaMemcpyAsync(&ns0, psweep_ns, sizeof(ns0), cudaMemcpyDeviceToHost, stream));
      int64_t k = h_iter;
      bool f = h_folded;
      double bsum = 0;
      const double cells = static_cast<double>(m) * static_cast<double>(n);
      for (int64_t it = 0; it < n_iters; ++it, ++k) {
        int md;
        bool fa;
        RC_TRY(pass_mode(k, f, &md, &fa));
        f = fa;
        bsum += (md == kSkip ? 2.0 : 3.0) * sizeof(T) * cells;
      }
      CUDA_TRY(cudaEventRecord(tev[0], stream));
      RC_TRY(launch_persist(n_iters));
      CUDA_TRY(cudaEventRecord(tev[1], stream));
      CUDA_TRY(cudaEventSynchronize(tev[1]));
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpy(&ns1, psweep_ns, sizeof(ns1), cudaMemcpyDeviceToHost));
      float ms = 0;
      CUDA_TRY(cudaEventElapsedTime(&ms, tev[0], tev[1]));
      if (total_ms) *total_ms = ms;
      if (pass_ms) *pass_ms = static_cast<double>(ns1 - ns0) * 1e-6;
      if (n_pass) *n_pass = n_iters;
      if (pass_bytes) *pass_bytes = bsum;
      if (launches) *launches = kernel_launch_count() - before;
      return 0;
    }
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

  int64_t batch_iters() const {
    // ~1 ms of pass traffic per batch at ~6 TB/s, at least 8 iterations
    const double bytes = 3.0 * sizeof(T) * static_cast<double>(m) * n;
    const double t_iter = bytes / 6.0e12 + (persist ? 6e-6 : 20e-6);
    int64_t bi = static_cast<int64_t>(1e-3 / t_iter) + 1;
    bi = std::max<int64_t>(8, std::min<int64_t>(bi, persist ? 1024 : 256));
    return bi + (bi & 1);
  }

  // Runs the loop until the device raises its stop flag (converged,
  // max_iters, numerical failure).  The host polls one batch behind so the
  // GPU queue never drains.
  // Sharded confirm after a gate pause (stop == 2): the exact report's sums
  // over all ranks, then the replicated decision (stop -> 1 or back to 0).
  // p2p shards: the last iteration's exact dual value / trace terms (the
  // row part is summed over the ranks, the column part is replicated)
  int shard_patch_pending() {
    TailArgs<T> ta = tail_args(h_iter, kFold, h_folded, true);
    launch_shard_pending_local<T>(ta, tdpart, tgrid, dpack, stream);
    RC_TRY(allreduce(dpack, 4, ncclSum));
    launch_shard_pending_patch<T>(ta, tdpart, tgrid, dpack, stream);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }

  int sharded_report(bool always) {
    if (xmode == 1) RC_TRY(shard_patch_pending());
    Book<T> hb;
    RC_TRY(read_book(&hb));
    TailArgs<T> ta = tail_args(hb.iter, kPlain0, hb.folded != 0, true);
    launch_report<T>(X, C, ta, false, always, stream);
    RC_TRY(allreduce(dpack + 4, 2, ncclSum));
    launch_report_final<T>(ta, always, stream);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }

  int run_sharded() {
    const int64_t bi = batch_iters();
    const int64_t limit = std::max<int64_t>(cfg.max_iters, 0) + 4 * bi + 4;
    int64_t guard = 0;
    while (true) {
      RC_TRY(enqueue(bi));
      Book<T> hb;
      RC_TRY(read_book(&hb));
      if (hb.stop == 2) {
        RC_TRY(sharded_report(false));
        RC_TRY(read_book(&hb));
      }
      h_iter = hb.iter;  // the batch may have run past a pause: resync
      h_folded = hb.folded != 0;
      if (hb.stop == 1) break;
      if ((guard += bi) > limit) break;
    }
    return 0;
  }

  int run() {
    if (!initialized) return set_error(DROTB_ERRC_BAD_CONFIG, "session not initialized");
    if (sharded) return run_sharded();
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
  int finalize_pending() {  // coop tail: patch the last iteration's exact dual / trace terms
    if (fiter) {  // single-launch iteration: materialize pending duals + patch
      launch_iter_finalize<T>(iter_args(h_iter, kFold, h_folded), stream);
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
    if (!coop || !tdpart) return 0;
    if (sharded) return xmode == 1 ? shard_patch_pending() : 0;
    TailArgs<T> ta = tail_args(h_iter, kFold, h_folded, true);
    launch_tail_finalize<T>(ta, tdpart, tgrid, stream);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }

  int finish(int32_t* status, int64_t* iterations, drotb_report* rep) {
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
  int get_plan(T* plan, T* mu, T* nu) {
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
  int support(double rel_tau, double abs_tau, int64_t* nnz, double* xmax) {
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

  int get_trace(drotb_trace_row* out, int64_t cap, int64_t* len) {
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

  // ---- external-state single step (drot_step, solver.hpp:361-370) --------
  int load_state(const T* xy, int32_t folded, const T* rs, const T* cs,
                 const T* ya, const T* yb, T alpha, const T* r, const T* s,
                 T beta, int64_t iter) {
    RC_TRY(resolve_rho());
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
    hb.phi_mat = 1;
    CUDA_TRY(cudaMemcpyAsync(book, &hb, sizeof(hb), cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    want_dual = false;  // default PassOptions (solver.hpp:367)
    want_dx = false;
    gate = false;
    h_iter = iter;
    h_folded = folded != 0;
    h_stale = false;
    initialized = true;
    return 0;
  }

  int store_state(T* xy, int32_t* folded, T* rs, T* cs, T* ya, T* yb, T* alpha,
                  T* r, T* s, T* beta, int64_t* iter, bool full) {
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
  int engine_pass(T* xy, const T* cost, const T* rs, const T* cs, T rho_,
                  int mode, bool dual, bool dx, bool deterministic, T* row_sums,
                  T* col_sums, drotb_pass_out* out) {
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
};

template <class T>
static Session<T>* as_session(void* s) {
  return static_cast<Session<T>*>(s);
}

}  // namespace drotb

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using drotb::Session;

struct drotb_session {
  int32_t precision;
  void* impl;
};
struct drotb_engine {
  int32_t precision;
  void* impl;
};

namespace {

int guard_exceptions(const std::exception& e) {
  return drotb::set_cuda_error(DROTB_ERR_CUDA, std::string("exception: ") + e.what());
}

drotb_config effective(const drotb_config* cfg) {
  drotb_config c;
  drotb_config_default(&c);
  if (cfg) c = *cfg;
  return c;
}

// One cached session per host thread and precision: a repeated solve of the
// same shape and configuration reuses its device buffers, stream, schedule
// and captured graphs instead of reallocating ~2*m*n*sizeof(T) per call
// (drotb_release_cache() frees it).
template <class T>
struct SolveCache {
  std::unique_ptr<Session<T>> s;
  int64_t m = 0, n = 0;
  drotb_config cfg{};
  Session<T>* get(int64_t m_, int64_t n_, const drotb_config& c, int* rc) {
    *rc = 0;
    if (s && m == m_ && n == n_ && std::memcmp(&cfg, &c, sizeof(c)) == 0) return s.get();
    s.reset();  // free the old buffers before allocating new ones
    std::unique_ptr<Session<T>> fresh(new Session<T>());
    *rc = fresh->create(m_, n_, c);
    if (*rc) return nullptr;
    s = std::move(fresh);
    m = m_;
    n = n_;
    cfg = c;
    return s.get();
  }
};
template <class T>
static SolveCache<T>& solve_cache() {
  static thread_local SolveCache<T> c;
  return c;
}

template <class T>
int solve_t(const T* C, int64_t m, int64_t n, const T* p, const T* q,
            const drotb_config* cfgp, const T* x0, T* plan, T* mu, T* nu,
            T* rho_out, drotb_report* rep, drotb_trace_row* trace,
            int64_t trace_cap, int64_t* trace_len, int64_t* iters,
            int32_t* status, double* wall) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  drotb::clear_error();
  const drotb_config cfg = effective(cfgp);
  try {
    if (m <= 0 || n <= 0)
      return drotb::set_error(DROTB_ERRC_EMPTY_DIMENSION, "cost matrix has an empty dimension");
    int crc = 0;
    Session<T>* s = solve_cache<T>().get(m, n, cfg, &crc);
    if (!s) return crc;
    RC_TRY(s->set_problem(C, p, q, false, true));
    RC_TRY(s->init(x0));
    RC_TRY(s->run());
    const auto t1 = clk::now();
    RC_TRY(s->finish(status, iters, rep));
    RC_TRY(s->get_plan(plan, mu, nu));
    RC_TRY(s->get_trace(trace, trace_cap, trace_len));
    if (rho_out) *rho_out = s->rho;
    if (wall) *wall = std::chrono::duration<double>(t1 - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

template <class T>
int step_t(T* xy, int32_t* folded, T* rs, T* cs, T* ya, T* yb, T* alpha, T* r,
           T* s, T* beta, int64_t* iter, const T* C, int64_t m, int64_t n,
           const T* p, const T* q, const drotb_config* cfgp) {
  drotb::clear_error();
  const drotb_config cfg = effective(cfgp);
  try {
    std::unique_ptr<Session<T>> ss(new Session<T>());
    RC_TRY(ss->create(m, n, cfg));
    RC_TRY(ss->set_problem(C, p, q, false, false));
    RC_TRY(ss->load_state(xy, *folded, rs, cs, ya, yb, *alpha, r, s, *beta, *iter));
    RC_TRY(ss->enqueue_iteration());
    CUDA_TRY(cudaGetLastError());
    drotb::Book<T> hb;
    RC_TRY(ss->read_book(&hb));
    if (hb.pass_bad) {
      RC_TRY(ss->store_state(xy, folded, rs, cs, ya, yb, alpha, r, s, beta, iter, false));
      return drotb::set_error(DROTB_ERRC_NON_FINITE_ITERATE,
                              "non-finite value in iterate update");
    }
    return ss->store_state(xy, folded, rs, cs, ya, yb, alpha, r, s, beta, iter, true);
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

template <class T>
int init_state_t(T* xy, int32_t* folded, T* rs, T* cs, T* ya, T* yb, T* alpha,
                 T* r, T* s, T* beta, int64_t* iter, const T* C, int64_t m,
                 int64_t n, const T* p, const T* q, const T* x0,
                 const drotb_config* cfgp) {
  drotb::clear_error();
  drotb_config cfg = effective(cfgp);
  try {
    std::unique_ptr<Session<T>> ss(new Session<T>());
    RC_TRY(ss->create(m, n, cfg));
    RC_TRY(ss->set_problem(C, p, q, false, false));
    RC_TRY(ss->init(x0));
    return ss->store_state(xy, folded, rs, cs, ya, yb, alpha, r, s, beta, iter, true);
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

template <class T>
int engine_pass_t(drotb_engine* eng, T* xy, const T* C, const T* rs,
                  const T* cs, T rho, int32_t kind, int32_t fold,
                  int32_t* cost_folded, int32_t parity, int32_t want_dual,
                  int32_t want_dx, int32_t deterministic, T* row_sums,
                  T* col_sums, drotb_pass_out* out, drotb_counters* counters) {
  drotb::clear_error();
  if (!eng) return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "null engine");
  if ((eng->precision == 0) != (sizeof(T) == 4))
    return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "engine precision mismatch");
  auto* s = static_cast<Session<T>*>(eng->impl);
  int mode;
  bool fold_write = false;
  if (kind == DROTB_PASS_SKIP_COST) {
    if (!cost_folded) return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "cost_folded required");
    if ((fold != 0) == (*cost_folded != 0))
      return drotb::set_error(DROTB_ERRC_FOLD_STATE_MISMATCH,
                              fold ? "array already stores X - rho C"
                                   : "array does not store X - rho C");
    mode = fold ? drotb::kFold : drotb::kSkip;
    fold_write = fold != 0;
  } else {
    mode = parity ? drotb::kPlain1 : drotb::kPlain0;
  }
  try {
    const bool dual = want_dual != 0;
    const bool dx = want_dx != 0;
    RC_TRY(s->engine_pass(xy, C, rs, cs, rho, mode, dual, dx, deterministic != 0,
                          row_sums, col_sums, out));
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
  if (kind == DROTB_PASS_SKIP_COST) *cost_folded = fold_write ? 1 : 0;
  if (kind == DROTB_PASS_UNFUSED && out) {
    out->dual_valid = want_dual != 0;
    out->dx_valid = want_dx != 0;
  }
  if (counters) {  // MemoryCounters (fused.hpp:305-310, 423-519)
    const uint64_t cells = static_cast<uint64_t>(s->m) * static_cast<uint64_t>(s->n);
    counters->passes += 1;
    if (kind == DROTB_PASS_UNFUSED) {
      counters->xy_elems_read += 4 * cells;
      counters->xy_elems_written += cells;
      counters->cost_elems_read += 2 * cells;
    } else {
      counters->xy_elems_read += cells;
      counters->xy_elems_written += cells;
      if (mode != drotb::kSkip) counters->cost_elems_read += cells;
    }
  }
  return 0;
}

template <class T>
int check_problem_t(const T* C, int64_t m, int64_t n, const T* p, const T* q) {
  drotb::clear_error();
  drotb_config cfg;
  drotb_config_default(&cfg);
  try {
    std::unique_ptr<Session<T>> s(new Session<T>());
    RC_TRY(s->create(m, n, cfg));
    return s->set_problem(C, p, q, false, true);
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

}  // namespace

// Marginals of the generated instances (rank-local slice of p, all of q).
//   0 uniform 1/m (gen_gaussian_problem, probgen.hpp:163-164)
//   1 dyadic-exact uniform (passes the 1e-12 check in fp32)
//   2 Dirichlet(1..1) (probgen.hpp:115-127, substreams 4 and 5)
//   3 random_simplex(seed ^ 0x1111), random_simplex(seed ^ 0x2222)
//     (oracles.hpp:137-147, the pattern of test_reference.cpp:22-29)
namespace drotb {
template <class T>
static int gen_marginals(int64_t mg, int64_t n, uint64_t seed, int32_t kind,
                         std::vector<T>& pg, std::vector<T>& q) {
  pg.assign(static_cast<size_t>(mg), T(0));
  q.assign(static_cast<size_t>(n), T(0));
  if (kind == 1) {
    RC_TRY(dyadic_marginal<T>(mg, pg.data()));
    RC_TRY(dyadic_marginal<T>(n, q.data()));
  } else if (kind == 2 || kind == 3) {
    std::vector<double> pd(static_cast<size_t>(mg)), qd(static_cast<size_t>(n));
    if (kind == 2) {
      dirichlet_marginal(seed, 4, mg, pd.data());
      dirichlet_marginal(seed, 5, n, qd.data());
    } else {
      random_simplex(mg, seed ^ 0x1111u, pd.data());
      random_simplex(n, seed ^ 0x2222u, qd.data());
    }
    for (int64_t i = 0; i < mg; ++i) pg[i] = static_cast<T>(pd[i]);
    for (int64_t j = 0; j < n; ++j) q[j] = static_cast<T>(qd[j]);
  } else if (kind == 0) {
    for (int64_t i = 0; i < mg; ++i) pg[i] = static_cast<T>(1.0 / static_cast<double>(mg));
    for (int64_t j = 0; j < n; ++j) q[j] = static_cast<T>(1.0 / static_cast<double>(n));
  } else {
    return set_error(DROTB_ERRC_BAD_CONFIG, "unknown marginal kind");
  }
  return 0;
}
}  // namespace drotb

// residual_report (problem.hpp:174-225) on the device: transient buffers,
// host in/out.
template <class T>
static int residual_report_t(const T* C, int64_t m, int64_t n, const T* p, const T* q,
                             const T* plan, const T* mu, const T* nu, int32_t exact,
                             drotb_report* out) {
  if (m <= 0 || n <= 0)
    return drotb::set_error(DROTB_ERRC_EMPTY_DIMENSION, "residual_report: empty dimension");
  if (!C || !p || !q || !plan || !mu || !nu || !out)
    return drotb::set_error(DROTB_ERRC_SHAPE_MISMATCH, "residual_report: null argument");
  const size_t mn = static_cast<size_t>(m) * static_cast<size_t>(n);
  // scratch: rowdev[m], coldev[n], colobj[n], coldsq[n] (report.cu), then out[4]
  const size_t ns = static_cast<size_t>(m) + 3 * static_cast<size_t>(n);
  const size_t tb = (sizeof(T) * (2 * mn + 2 * static_cast<size_t>(m + n)) + 15) & ~size_t{15};
  const size_t db = sizeof(double) * (ns + 4);
  char* buf = nullptr;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&buf), tb + db));
  std::unique_ptr<char, decltype(&cudaFree)> hold(buf, &cudaFree);
  T* dX = reinterpret_cast<T*>(buf);
  T* dC = dX + mn;
  T* dmu = dC + mn;
  T* dp = dmu + m;
  T* dnu = dp + m;
  T* dq = dnu + n;
  double* scratch = reinterpret_cast<double*>(buf + tb);
  double* dout = scratch + ns;
  CUDA_TRY(cudaMemcpy(dX, plan, sizeof(T) * mn, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dC, C, sizeof(T) * mn, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dmu, mu, sizeof(T) * m, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dp, p, sizeof(T) * m, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dnu, nu, sizeof(T) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dq, q, sizeof(T) * n, cudaMemcpyHostToDevice));
  drotb::launch_residual_report<T>(dX, dC, dmu, dnu, dp, dq, m, n, exact != 0, scratch, dout,
                                   nullptr);
  CUDA_TRY(cudaGetLastError());
  double r[4];
  CUDA_TRY(cudaMemcpy(r, dout, sizeof(r), cudaMemcpyDeviceToHost));
  out->r_primal = r[0];
  out->r_dual = r[1];
  out->gap = r[2];
  out->objective = r[3];
  return 0;
}

extern "C" {

int32_t drotb_abi_version(void) { return DROTB_ABI_VERSION; }
const char* drotb_last_error(void) { return drotb::last_error_cstr(); }
const char* drotb_errc_name(int32_t errc) { return drotb::errc_name(errc); }
int64_t drotb_kernel_launches(void) { return drotb::kernel_launch_count(); }

void drotb_config_default(drotb_config* c) {  // DrotConfig{} (solver.hpp:51-88)
  std::memset(c, 0, sizeof(*c));
  c->rho0 = 2.0;
  c->has_rho_override = 0;
  c->relative_tolerances = 0;
  c->rho_override = 0.0;
  c->tol_primal = c->tol_dual = c->tol_gap = 1e-4;
  c->max_iters = 100000;
  c->check_every = 1;
  c->engine = DROTB_ENGINE_FUSED;
  c->skip_cost = 1;
  c->deterministic = 1;
  c->record_trace = 1;
  c->workers = 0;
  c->block_rows = 64;
  c->work_size = 4;
  c->trace_every = 1;
  c->precision = 1;
  c->device = -1;
  c->order = DROTB_ORDER_FAST;
  c->use_graphs = 1;
}

int drotb_solve_f32(const float* C, int64_t m, int64_t n, const float* p,
                    const float* q, const drotb_config* cfg, const float* x0,
                    float* plan, float* mu, float* nu, float* rho_out,
                    drotb_report* rep, drotb_trace_row* trace,
                    int64_t trace_cap, int64_t* trace_len, int64_t* iters,
                    int32_t* status, double* wall) {
  return solve_t<float>(C, m, n, p, q, cfg, x0, plan, mu, nu, rho_out, rep,
                        trace, trace_cap, trace_len, iters, status, wall);
}
int drotb_solve_f64(const double* C, int64_t m, int64_t n, const double* p,
                    const double* q, const drotb_config* cfg, const double* x0,
                    double* plan, double* mu, double* nu, double* rho_out,
                    drotb_report* rep, drotb_trace_row* trace,
                    int64_t trace_cap, int64_t* trace_len, int64_t* iters,
                    int32_t* status, double* wall) {
  return solve_t<double>(C, m, n, p, q, cfg, x0, plan, mu, nu, rho_out, rep,
                         trace, trace_cap, trace_len, iters, status, wall);
}

int drotb_step_f32(float* xy, int32_t* folded, float* rs, float* cs, float* ya,
                   float* yb, float* alpha, float* r, float* s, float* beta,
                   int64_t* iter, const float* C, int64_t m, int64_t n,
                   const float* p, const float* q, const drotb_config* cfg) {
  return step_t<float>(xy, folded, rs, cs, ya, yb, alpha, r, s, beta, iter, C,
                       m, n, p, q, cfg);
}
int drotb_step_f64(double* xy, int32_t* folded, double* rs, double* cs,
                   double* ya, double* yb, double* alpha, double* r, double* s,
                   double* beta, int64_t* iter, const double* C, int64_t m,
                   int64_t n, const double* p, const double* q,
                   const drotb_config* cfg) {
  return step_t<double>(xy, folded, rs, cs, ya, yb, alpha, r, s, beta, iter, C,
                        m, n, p, q, cfg);
}
int drotb_init_state_f32(float* xy, int32_t* folded, float* rs, float* cs,
                         float* ya, float* yb, float* alpha, float* r, float* s,
                         float* beta, int64_t* iter, const float* C, int64_t m,
                         int64_t n, const float* p, const float* q,
                         const float* x0, const drotb_config* cfg) {
  return init_state_t<float>(xy, folded, rs, cs, ya, yb, alpha, r, s, beta,
                             iter, C, m, n, p, q, x0, cfg);
}
int drotb_init_state_f64(double* xy, int32_t* folded, double* rs, double* cs,
                         double* ya, double* yb, double* alpha, double* r,
                         double* s, double* beta, int64_t* iter,
                         const double* C, int64_t m, int64_t n, const double* p,
                         const double* q, const double* x0,
                         const drotb_config* cfg) {
  return init_state_t<double>(xy, folded, rs, cs, ya, yb, alpha, r, s, beta,
                              iter, C, m, n, p, q, x0, cfg);
}

int drotb_engine_create(drotb_engine** eng, int64_t m, int64_t n,
                        int64_t block_rows, int64_t work_size,
                        int32_t precision, int32_t device) {
  drotb::clear_error();
  *eng = nullptr;
  drotb_config cfg;
  drotb_config_default(&cfg);
  cfg.block_rows = block_rows;
  cfg.work_size = work_size;
  cfg.device = device;
  cfg.order = DROTB_ORDER_FAST;
  try {
    std::unique_ptr<drotb_engine> e(new drotb_engine{precision, nullptr});
    if (precision == 0) {
      std::unique_ptr<Session<float>> s(new Session<float>());
      RC_TRY(s->create(m, n, cfg, true));
      e->impl = s.release();
    } else {
      std::unique_ptr<Session<double>> s(new Session<double>());
      RC_TRY(s->create(m, n, cfg, true));
      e->impl = s.release();
    }
    *eng = e.release();
    return 0;
  } catch (const std::exception& ex) {
    return guard_exceptions(ex);
  }
}

void drotb_engine_destroy(drotb_engine* eng) {
  if (!eng) return;
  if (eng->precision == 0)
    delete static_cast<Session<float>*>(eng->impl);
  else
    delete static_cast<Session<double>*>(eng->impl);
  delete eng;
}

int drotb_engine_pass_f32(drotb_engine* eng, float* xy, const float* C,
                          const float* rs, const float* cs, float rho,
                          int32_t kind, int32_t fold, int32_t* cost_folded,
                          int32_t parity, int32_t want_dual, int32_t want_dx,
                          int32_t deterministic, float* row_sums,
                          float* col_sums, drotb_pass_out* out,
                          drotb_counters* counters) {
  return engine_pass_t<float>(eng, xy, C, rs, cs, rho, kind, fold, cost_folded,
                              parity, want_dual, want_dx, deterministic,
                              row_sums, col_sums, out, counters);
}
int drotb_engine_pass_f64(drotb_engine* eng, double* xy, const double* C,
                          const double* rs, const double* cs, double rho,
                          int32_t kind, int32_t fold, int32_t* cost_folded,
                          int32_t parity, int32_t want_dual, int32_t want_dx,
                          int32_t deterministic, double* row_sums,
                          double* col_sums, drotb_pass_out* out,
                          drotb_counters* counters) {
  return engine_pass_t<double>(eng, xy, C, rs, cs, rho, kind, fold,
                               cost_folded, parity, want_dual, want_dx,
                               deterministic, row_sums, col_sums, out,
                               counters);
}

int drotb_check_problem_f32(const float* C, int64_t m, int64_t n,
                            const float* p, const float* q) {
  return check_problem_t<float>(C, m, n, p, q);
}
int drotb_check_problem_f64(const double* C, int64_t m, int64_t n,
                            const double* p, const double* q) {
  return check_problem_t<double>(C, m, n, p, q);
}

// ---- sessions ----------------------------------------------------------------
#define DROTB_DISPATCH(s, call)                                  \
  ((s)->precision == 0 ? drotb::as_session<float>((s)->impl)->call \
                       : drotb::as_session<double>((s)->impl)->call)

int drotb_session_create(drotb_session** s, int64_t m, int64_t n,
                         int32_t precision, const drotb_config* cfgp) {
  drotb::clear_error();
  *s = nullptr;
  const drotb_config cfg = effective(cfgp);
  try {
    std::unique_ptr<drotb_session> h(new drotb_session{precision, nullptr});
    if (precision == 0) {
      std::unique_ptr<Session<float>> ss(new Session<float>());
      RC_TRY(ss->create(m, n, cfg));
      h->impl = ss.release();
    } else {
      std::unique_ptr<Session<double>> ss(new Session<double>());
      RC_TRY(ss->create(m, n, cfg));
      h->impl = ss.release();
    }
    *s = h.release();
    return 0;
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

void drotb_session_destroy(drotb_session* s) {
  if (!s) return;
  if (s->precision == 0)
    delete drotb::as_session<float>(s->impl);
  else
    delete drotb::as_session<double>(s->impl);
  delete s;
}

int drotb_session_set_stream(drotb_session* s, void* stream) {
  drotb::clear_error();
  return DROTB_DISPATCH(s, set_stream(stream));
}

int drotb_session_set_problem(drotb_session* s, const void* C, const void* p,
                              const void* q, int32_t is_device) {
  drotb::clear_error();
  if (s->precision == 0)
    return drotb::as_session<float>(s->impl)->set_problem(
        static_cast<const float*>(C), static_cast<const float*>(p),
        static_cast<const float*>(q), is_device != 0, true);
  return drotb::as_session<double>(s->impl)->set_problem(
      static_cast<const double*>(C), static_cast<const double*>(p),
      static_cast<const double*>(q), is_device != 0, true);
}

// K7: the Gaussian instance generated on the device (probgen.cu); only the
// O(m+n) points and marginals are drawn on the host.
int drotb_session_gen_gaussian(drotb_session* s, double sigma_t, uint64_t seed,
                               int32_t marginals) {
  drotb::clear_error();
  auto go = [&](auto* ss) -> int {
    using T = typename std::remove_pointer<decltype(ss->X)>::type;
    const int64_t m = ss->m, n = ss->n, mg = ss->m_global, r0 = ss->row_begin;
    std::vector<double> xs, xt;
    RC_TRY(drotb::gaussian_points(mg, n, sigma_t, seed, xs, xt));
    double* dpts = nullptr;
    unsigned long long* dmax = nullptr;
    // stream-ordered allocation: no device-wide synchronization (shards of one
    // process may be spinning in a collective on the same device)
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dpts), sizeof(double) * 2 * (mg + n) + 16,
                             ss->stream));
    cudaStream_t hs = ss->stream;
    auto freer = [hs](double* ptr) { cudaFreeAsync(ptr, hs); };
    std::unique_ptr<double, decltype(freer)> hold(dpts, freer);
    dmax = reinterpret_cast<unsigned long long*>(dpts + 2 * (mg + n));
    double* dxs = dpts;
    double* dxt = dpts + 2 * mg;
    CUDA_TRY(cudaMemcpyAsync(dxs, xs.data(), sizeof(double) * 2 * mg, cudaMemcpyHostToDevice,
                             ss->stream));
    CUDA_TRY(cudaMemcpyAsync(dxt, xt.data(), sizeof(double) * 2 * n, cudaMemcpyHostToDevice,
                             ss->stream));
    drotb::launch_gaussian_cmax(dxs, dxt, mg, n, dmax, ss->stream);
    unsigned long long bits = 0;
    CUDA_TRY(cudaMemcpyAsync(&bits, dmax, sizeof(bits), cudaMemcpyDeviceToHost, ss->stream));
    CUDA_TRY(cudaStreamSynchronize(ss->stream));
    double cmax;
    std::memcpy(&cmax, &bits, sizeof(cmax));
    if (!(cmax > 0)) return drotb::set_error(DROTB_ERRC_DEGENERATE_COST, "all samples coincide");
    drotb::launch_gaussian_cost<T>(dxs + 2 * r0, dxt, m, n, ss->ld, dmax, ss->C, ss->stream);
    CUDA_TRY(cudaGetLastError());
    std::vector<T> pg, q;
    RC_TRY(drotb::gen_marginals<T>(mg, n, seed, marginals, pg, q));
    RC_TRY(ss->set_problem(nullptr, pg.data() + r0, q.data(), false, true));
    return 0;
  };
  try {
    if (s->precision == 0) return go(drotb::as_session<float>(s->impl));
    return go(drotb::as_session<double>(s->impl));
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

// K7: random_matrix(m, n, seed, lo, hi) (oracles.hpp:128-135) generated on
// the device, in the global storage order (shards generate their rows).
int drotb_session_gen_uniform(drotb_session* s, uint64_t seed, double lo, double hi,
                              int32_t marginals) {
  drotb::clear_error();
  auto go = [&](auto* ss) -> int {
    using T = typename std::remove_pointer<decltype(ss->X)>::type;
    const int64_t m = ss->m, n = ss->n, mg = ss->m_global, r0 = ss->row_begin;
    drotb::launch_uniform_cost<T>(seed, lo, hi, m, mg, r0, n, ss->ld, ss->C, ss->stream);
    CUDA_TRY(cudaGetLastError());
    std::vector<T> pg, q;
    RC_TRY(drotb::gen_marginals<T>(mg, n, seed, marginals, pg, q));
    RC_TRY(ss->set_problem(nullptr, pg.data() + r0, q.data(), false, true));
    return 0;
  };
  try {
    if (s->precision == 0) return go(drotb::as_session<float>(s->impl));
    return go(drotb::as_session<double>(s->impl));
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

int drotb_residual_report_f32(const float* C, int64_t m, int64_t n, const float* p,
                              const float* q, const float* plan, const float* mu,
                              const float* nu, int32_t exact, drotb_report* out) {
  drotb::clear_error();
  return residual_report_t<float>(C, m, n, p, q, plan, mu, nu, exact, out);
}
int drotb_residual_report_f64(const double* C, int64_t m, int64_t n, const double* p,
                              const double* q, const double* plan, const double* mu,
                              const double* nu, int32_t exact, drotb_report* out) {
  drotb::clear_error();
  return residual_report_t<double>(C, m, n, p, q, plan, mu, nu, exact, out);
}

void drotb_release_cache(void) {
  solve_cache<float>().s.reset();
  solve_cache<double>().s.reset();
}

// Profiling aid: copy (and reset) the 8 tail-phase timestamps (ns).
int drotb_session_tail_stamps(drotb_session* s, uint64_t* out8) {
  auto go = [&](auto* ss) -> int {
    if (!ss->tstamps) return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "DROTB_TAIL_STAMPS not set");
    CUDA_TRY(cudaStreamSynchronize(ss->stream));
    CUDA_TRY(cudaMemcpy(out8, ss->tstamps, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    uint64_t init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
    CUDA_TRY(cudaMemcpy(ss->tstamps, init, sizeof(init), cudaMemcpyHostToDevice));
    return 0;
  };
  if (s->precision == 0) return go(drotb::as_session<float>(s->impl));
  return go(drotb::as_session<double>(s->impl));
}

// Debug aid: device addresses of the book, the tail barrier words and the
// exchange buffer (for side-stream inspection of a stuck exchange).
int drotb_session_debug_ptrs(drotb_session* s, uint64_t* out4) {
  auto go = [&](auto* ss) -> int {
    out4[0] = reinterpret_cast<uint64_t>(ss->book);
    out4[1] = reinterpret_cast<uint64_t>(ss->tbar);
    out4[2] = reinterpret_cast<uint64_t>(ss->xbuf);
    out4[3] = static_cast<uint64_t>(ss->tgrid);
    return 0;
  };
  if (s->precision == 0) return go(drotb::as_session<float>(s->impl));
  return go(drotb::as_session<double>(s->impl));
}

int32_t drotb_session_persistent_grid(drotb_session* s) {
  if (s->precision == 0) {
    auto* ss = drotb::as_session<float>(s->impl);
    return ss->persist ? ss->pgrid : 0;
  }
  auto* ss = drotb::as_session<double>(s->impl);
  return ss->persist ? ss->pgrid : 0;
}

int drotb_session_support(drotb_session* s, double rel_tau, double abs_tau, int64_t* nnz,
                          double* xmax) {
  drotb::clear_error();
  try {
    return DROTB_DISPATCH(s, support(rel_tau, abs_tau, nnz, xmax));
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

// Download the session's (local) cost matrix, column-major m x n (tests of
// the on-device generator; the solver never needs it on the host).
int drotb_session_get_cost(drotb_session* s, void* out) {
  drotb::clear_error();
  if (s->precision == 0) {
    auto* ss = drotb::as_session<float>(s->impl);
    return ss->download_matrix(static_cast<float*>(out), ss->C);
  }
  auto* ss = drotb::as_session<double>(s->impl);
  return ss->download_matrix(static_cast<double*>(out), ss->C);
}

int drotb_session_init(drotb_session* s, const void* x0) {
  drotb::clear_error();
  if (s->precision == 0)
    return drotb::as_session<float>(s->impl)->init(static_cast<const float*>(x0));
  return drotb::as_session<double>(s->impl)->init(static_cast<const double*>(x0));
}

int drotb_session_enqueue(drotb_session* s, int64_t n_iters) {
  drotb::clear_error();
  return DROTB_DISPATCH(s, enqueue(n_iters));
}

int drotb_session_run(drotb_session* s) {
  drotb::clear_error();
  return DROTB_DISPATCH(s, run());
}

int drotb_session_synchronize(drotb_session* s) {
  drotb::clear_error();
  void* st = DROTB_DISPATCH(s, stream);
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(st)));
  return 0;
}

int drotb_session_status(drotb_session* s, int32_t* status, int64_t* iterations,
                         drotb_report* report) {
  drotb::clear_error();
  return DROTB_DISPATCH(s, finish(status, iterations, report));
}

int drotb_session_get_plan(drotb_session* s, void* plan, void* mu, void* nu) {
  drotb::clear_error();
  if (s->precision == 0)
    return drotb::as_session<float>(s->impl)->get_plan(
        static_cast<float*>(plan), static_cast<float*>(mu), static_cast<float*>(nu));
  return drotb::as_session<double>(s->impl)->get_plan(
      static_cast<double*>(plan), static_cast<double*>(mu), static_cast<double*>(nu));
}

void* drotb_session_device_xy(drotb_session* s) {
  return s->precision == 0 ? static_cast<void*>(drotb::as_session<float>(s->impl)->X)
                           : static_cast<void*>(drotb::as_session<double>(s->impl)->X);
}

void* drotb_session_stream(drotb_session* s) {
  return s->precision == 0 ? static_cast<void*>(drotb::as_session<float>(s->impl)->stream)
                           : static_cast<void*>(drotb::as_session<double>(s->impl)->stream);
}

int drotb_session_pass_bytes(drotb_session* s, double* bytes_fold,
                             double* bytes_skip) {
  const double cells = s->precision == 0
                           ? static_cast<double>(drotb::as_session<float>(s->impl)->m) *
                                 drotb::as_session<float>(s->impl)->n
                           : static_cast<double>(drotb::as_session<double>(s->impl)->m) *
                                 drotb::as_session<double>(s->impl)->n;
  const double sz = s->precision == 0 ? 4.0 : 8.0;
  if (bytes_fold) *bytes_fold = 3.0 * sz * cells;  // read X, C; write X
  if (bytes_skip) *bytes_skip = 2.0 * sz * cells;  // read X; write X
  return 0;
}

int drotb_session_run_timed(drotb_session* s, int64_t n_iters, double* total_ms,
                            double* pass_ms, int64_t* n_pass, double* pass_bytes,
                            int64_t* launches) {
  drotb::clear_error();
  return DROTB_DISPATCH(s, run_timed(n_iters, total_ms, pass_ms, n_pass, pass_bytes, launches));
}

int drotb_nccl_unique_id(char* out128) {
  drotb::clear_error();
  if (!drotb::nccl().ok)
    return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "NCCL unavailable: " + drotb::nccl().err);
  ncclUniqueId id;
  NCCL_TRY(drotb::nccl().getUniqueId(&id));
  static_assert(sizeof(id) == DROTB_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

int drotb_session_create_sharded(drotb_session** s, int64_t m_global, int64_t n,
                                 int32_t precision, const drotb_config* cfgp, int32_t rank,
                                 int32_t world_size, const char* nccl_id128,
                                 int64_t row_begin, int64_t row_end) {
  drotb::clear_error();
  *s = nullptr;
  const drotb_config cfg = effective(cfgp);
  try {
    std::unique_ptr<drotb_session> h(new drotb_session{precision, nullptr});
    if (precision == 0) {
      std::unique_ptr<Session<float>> ss(new Session<float>());
      RC_TRY(ss->create_sharded(m_global, n, cfg, rank, world_size, nccl_id128, row_begin,
                                row_end));
      h->impl = ss.release();
    } else {
      std::unique_ptr<Session<double>> ss(new Session<double>());
      RC_TRY(ss->create_sharded(m_global, n, cfg, rank, world_size, nccl_id128, row_begin,
                                row_end));
      h->impl = ss.release();
    }
    *s = h.release();
    return 0;
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

int drotb_session_create_sharded_p2p(drotb_session** s, int64_t m_global, int64_t n,
                                     int32_t precision, const drotb_config* cfgp, int32_t rank,
                                     int32_t world_size, int64_t row_begin, int64_t row_end) {
  drotb::clear_error();
  *s = nullptr;
  const drotb_config cfg = effective(cfgp);
  try {
    std::unique_ptr<drotb_session> h(new drotb_session{precision, nullptr});
    if (precision == 0) {
      std::unique_ptr<Session<float>> ss(new Session<float>());
      RC_TRY(ss->create_sharded(m_global, n, cfg, rank, world_size, nullptr, row_begin, row_end,
                                1));
      h->impl = ss.release();
    } else {
      std::unique_ptr<Session<double>> ss(new Session<double>());
      RC_TRY(ss->create_sharded(m_global, n, cfg, rank, world_size, nullptr, row_begin, row_end,
                                1));
      h->impl = ss.release();
    }
    *s = h.release();
    return 0;
  } catch (const std::exception& e) {
    return guard_exceptions(e);
  }
}

int drotb_session_exchange_buffer(drotb_session* s, uint64_t* dev_ptr, char* ipc_handle64) {
  drotb::clear_error();
  auto go = [&](auto* ss) -> int {
    if (ss->xmode != 1 || !ss->xbuf)
      return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "session has no peer exchange");
    if (dev_ptr) *dev_ptr = reinterpret_cast<uint64_t>(ss->xbuf);
    if (ipc_handle64) {
      cudaIpcMemHandle_t h;
      CUDA_TRY(cudaIpcGetMemHandle(&h, ss->xbuf));
      std::memcpy(ipc_handle64, &h, 64);
    }
    return 0;
  };
  if (s->precision == 0) return go(drotb::as_session<float>(s->impl));
  return go(drotb::as_session<double>(s->impl));
}

int drotb_session_attach_peers(drotb_session* s, const uint64_t* dev_ptrs,
                               const char* ipc_handles) {
  drotb::clear_error();
  if (!dev_ptrs && !ipc_handles)
    return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "attach_peers: no pointers or handles");
  return DROTB_DISPATCH(s, attach_peers(dev_ptrs, ipc_handles));
}

int drotb_shard_rows(int64_t m, int32_t world_size, int32_t rank, int64_t* row_begin,
                     int64_t* row_end) {
  // contiguous row blocks aligned to the 64-row v blocks, as even as possible
  drotb::clear_error();
  if (world_size < 1 || rank < 0 || rank >= world_size || m < 1)
    return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "invalid shard request");
  const int64_t blocks = (m + 63) / 64;
  const int64_t b0 = blocks * rank / world_size, b1 = blocks * (rank + 1) / world_size;
  *row_begin = std::min<int64_t>(m, b0 * 64);
  *row_end = std::min<int64_t>(m, b1 * 64);
  return 0;
}

}  // extern "C"
