// session_shard.cu -- row-sharded sessions: rank r owns rows
// [row_begin, row_end) of X and C; the per-iteration exchange of the column
// sums and scalars runs either inside the cooperative tail over NVLink peer
// memory (xmode 1: the one tail kernel of tail.cu with world > 1 -- integer
// atomics into every rank's sums, bit-identical for any rank count) or as
// NCCL allreduces between
// per-launch kernels (xmode 0).
#include <dlfcn.h>

#include "session.hpp"

namespace drotb {

NcclApi& nccl() {
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


// Row shard [row_begin, row_end) of an m_global x n problem on `world`
// ranks (one process per GPU); collectives over NCCL.
template <class T>
int Session<T>::create_sharded(int64_t m_glob, int64_t n_, const drotb_config& c, int rk, int ws, const char* id128, int64_t r0, int64_t r1, int exchange) {
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
  sharded_create = true;  // the sharded tails are set up below
  tc_rows = m_glob;       // the one-GPU sweep tiles (rank-count-independent sums)
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
    // the iteration tail's cross-rank counters, exact sums and column sums
    xa.off_ctr = xsetup_off + 2 * world * xsetup_bytes;
    xa.off_acc = xa.off_ctr + 2 * 4 * 128;
    xa.off_vsum = xa.off_acc + 2 * kXaWords * 8;
    xa.vwords = sizeof(T) == 4 ? 1 : 2;
    xbytes = xa.off_vsum + 2 * static_cast<int64_t>(xa.vwords) * n * 8;
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&xbuf), static_cast<size_t>(xbytes)));
    CUDA_TRY(cudaMemset(xbuf, 0, static_cast<size_t>(xbytes)));
    if (!xacc || !fx_ok) return set_error(DROTB_ERRC_BAD_CONFIG, "exact sums unavailable");
    if (xacc_owned) cudaFree(xacc);
    xacc = reinterpret_cast<long long*>(xbuf + xa.off_acc);
    xacc_owned = false;
    RC_TRY(dev_alloc(&xloc, 2 * static_cast<size_t>(kXaWords)));
    CUDA_TRY(cudaMemset(xloc, 0, sizeof(long long) * 2 * kXaWords));
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
template <class T>
int Session<T>::attach_peers(const uint64_t* ptrs, const char* handles) {
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


template <class T>
template <class U>
int Session<T>::allreduce(U* buf, size_t count, ncclRedOp_t op) {
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
template <class T>
int Session<T>::agree(int local_rc, const std::string& local_msg) {
  if (!sharded) return local_rc;
  int32_t v = local_rc;
  RC_TRY(h2d_small(dint, &v, sizeof(v)));
  RC_TRY(allreduce(dint, 1, ncclMax));
  RC_TRY(d2h_small(&v, dint, sizeof(v)));
  if (v == 0) return 0;
  if (v != local_rc)
    set_error_text("rank " + std::to_string(rank) + ": another rank failed: " +
                   std::string(v < DROTB_ERR_CUDA ? errc_name(v - 1) : "device error"));
  else
    set_error_text(local_msg);
  return v;
}


// Sharded confirm after a gate pause (stop == 2, the NCCL exchange): the
// exact report's sums over all ranks, then the replicated decision (stop ->
// 1 or back to 0); also the final report of a max_iters run.
template <class T>
int Session<T>::sharded_report(bool always) {
  Book<T> hb;
  RC_TRY(read_book(&hb));
  TailArgs<T> ta = tail_args(hb.iter, kPlain0, hb.folded != 0, true);
  launch_report<T>(X, C, ta, false, always, stream);
  RC_TRY(allreduce(dpack + 4, 2, ncclSum));
  launch_report_final<T>(ta, always, stream);
  CUDA_TRY(cudaGetLastError());
  return 0;
}


template <class T>
int Session<T>::run_sharded() {
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

// explicit instantiations (the members defined in this file)
template int Session<float>::create_sharded(int64_t m_glob, int64_t n_, const drotb_config& c, int rk, int ws, const char* id128, int64_t r0, int64_t r1, int exchange);
template int Session<double>::create_sharded(int64_t m_glob, int64_t n_, const drotb_config& c, int rk, int ws, const char* id128, int64_t r0, int64_t r1, int exchange);
template int Session<float>::attach_peers(const uint64_t* ptrs, const char* handles);
template int Session<double>::attach_peers(const uint64_t* ptrs, const char* handles);
template int Session<float>::agree(int local_rc, const std::string& local_msg);
template int Session<double>::agree(int local_rc, const std::string& local_msg);
template int Session<float>::sharded_report(bool always);
template int Session<double>::sharded_report(bool always);
template int Session<float>::run_sharded();
template int Session<double>::run_sharded();
template int Session<float>::allreduce<float>(float* buf, size_t count, ncclRedOp_t op);
template int Session<float>::allreduce<double>(double* buf, size_t count, ncclRedOp_t op);
template int Session<float>::allreduce<int32_t>(int32_t* buf, size_t count, ncclRedOp_t op);
template int Session<double>::allreduce<float>(float* buf, size_t count, ncclRedOp_t op);
template int Session<double>::allreduce<double>(double* buf, size_t count, ncclRedOp_t op);
template int Session<double>::allreduce<int32_t>(int32_t* buf, size_t count, ncclRedOp_t op);

}  // namespace drotb
