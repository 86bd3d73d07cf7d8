// tail.cu -- KT: the per-iteration tail of the solve loop (fast reduction
// order, one GPU) as ONE cooperative kernel after the fused sweep K1.
//
//   A  merge      u_i = sum of the K1 row strips, v_j = sum of the 64-row
//                 column strips (fused.hpp:312-321), r = u - p, s = v - q
//                 (solver.hpp:269-272); per-CTA partials of sum r, |r|^2,
//                 |s|^2 and of a fixed slice of the K1 CTA scalars
//   -- reduce-barrier: the last CTA to arrive reduces the per-CTA partials in
//      CTA order and runs the scalar recursions (solver.hpp:273-277,
//      418-437) on the device Book, then releases the others --
//   B  update     phi, varphi, a, b (solver.hpp:279-289) + dual-value and
//                 fixed-point partials
//   -- reduce-barrier: last CTA -> gate (solver.hpp:443-504) --
//   C  report     only when the gate fired: the exact matched-pair report
//                 of (X_{k+1}, phi/rho, varphi/rho) (solver.hpp:312-354)
//   -- reduce-barrier: last CTA -> confirm decision (solver.hpp:508-519) --
//
// It replaces three kernels and a graph IF node of the per-launch tail
// (merge_kernel, update_kernel, report_kernel) whose launch gaps and
// single-block "last block" reductions cost ~32 us per iteration at 10k^2
// (r1 measurement).  The reduce-barrier makes the grid-wide reduction part of
// the barrier itself: no CTA re-reads all partials (a G^2 L2 hot spot) and no
// second barrier is needed to broadcast the totals.  Deterministic: every
// reduction runs in a fixed order independent of which CTA arrives last.
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "drotb_internal.hpp"
#include "sweep.cuh"
#include "gate.cuh"

namespace drotb {

namespace {

constexpr int kTT = 256;            // threads per CTA

// profiling aid (DROTB_TAIL_STAMPS): timeline points (drotb_internal.hpp)
#define TAIL_STAMP(pt)                                                          \
  do {                                                                          \
    if (t.stamps && threadIdx.x == 0) timeline_point(t.stamps, it_stamp, pt, global_ns()); \
  } while (0)

// Counter barrier of the cooperative tail: every CTA arrives with one
// release-add on the counter of this launch and spins (relaxed loads, no
// cache invalidation per poll) until all G arrivals are visible, then
// acquires.  No CTA waits for another to compute anything: after the
// barrier every CTA reduces the per-CTA partials itself, in the same fixed
// order, and runs the scalar logic on its own shared-memory copy of the Book
// (bit-identical everywhere); CTA 0 alone writes the Book and the trace.
// Counters: bar[kCtr0] / bar[kCtr1] by iteration parity; a launch resets the
// other parity's counter for the next launch (consecutive tails alternate).
constexpr int kCtr0 = 768, kCtr1 = 896;
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void count_barrier(unsigned* ctr, unsigned target,
                                              unsigned long long* stamps, int64_t it_stamp) {
  __syncthreads();  // this CTA's partials are written (CTA scope)
  if (threadIdx.x == 0) {
    red_release_add(ctr, 1u);
    while (static_cast<int>(ld_relaxed(ctr) - target) < 0) {
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (stamps) timeline_point(stamps, it_stamp, 10, global_ns());
  }
  __syncthreads();
}

template <class T>
__device__ __forceinline__ void book_store_cta0(Book<T>* dst, const Book<T>* src) {
  constexpr int W = static_cast<int>(sizeof(Book<T>) / 8);
  __syncthreads();
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k < W; k += blockDim.x)
      reinterpret_cast<unsigned long long*>(dst)[k] =
          reinterpret_cast<const unsigned long long*>(src)[k];
}

// update-phase threads: warps kUW.. (warps 0 and 1 run the scalar logic of
// barrier 1 meanwhile)
constexpr int kUW = 2;

// ---- row shards (TailArgs::x, world > 1) ----------------------------------
__device__ __forceinline__ void red_sys_u64(long long* p, long long v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_sys_max_u64(long long* p, long long v) {
  asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// this iteration's accumulators / counters / column sums of rank r
__device__ __forceinline__ long long* x_acc(const XArgs& x, int r, int par) {
  return reinterpret_cast<long long*>(x.peers[r] + x.off_acc) + par * kXaWords;
}
__device__ __forceinline__ unsigned* x_ctr(const XArgs& x, int r, int par, int b) {
  return reinterpret_cast<unsigned*>(x.peers[r] + x.off_ctr) + (par * 4 + b) * 32;
}
__device__ __forceinline__ long long* x_vsum(const XArgs& x, int r, int par, int64_t n) {
  return reinterpret_cast<long long*>(x.peers[r] + x.off_vsum) + par * n * x.vwords;
}
// cross-rank barrier b of this iteration: every CTA of every rank adds one to
// every rank's counter (release, system scope) and waits for world * G on its own
__device__ __forceinline__ void xrank_barrier(const XArgs& x, int par, int b, unsigned want,
                                              unsigned long long* stamps, int64_t it_stamp) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int r = 0; r < x.world; ++r) red_release_sys_u32(x_ctr(x, r, par, b), 1u);
    const unsigned* mine = x_ctr(x, x.rank, par, b);
    while (static_cast<int>(ld_relaxed_sys(mine) - want) < 0) {
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (stamps) timeline_point(stamps, it_stamp, 10, global_ns());
  }
  __syncthreads();
}

// red_cta_hilo with a destination per sum: sums whose bit is set in
// all_mask (row-side sums of this rank's rows) go to every rank's
// accumulator, the others (replicated column-side sums) to this rank's only
template <int NT, int K>
__device__ __forceinline__ void red_cta_hilo_x(HiLo (&v)[K], int word0, int all_mask,
                                               const XArgs& x, int par, long long* local,
                                               long long* sh) {
  constexpr int kTW = NT / 32;
  static_assert(K <= 8, "16 words per lane");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long w[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w[2 * k] = k < K ? v[k].hi : 0;
    w[2 * k + 1] = k < K ? v[k].lo : 0;
  }
  const long long ws = bfly16(w, lane);
  __syncthreads();
  if ((lane & 1) == 0) sh[bfly16_word(lane) * kTW + warp] = ws;
  __syncthreads();
  if (threadIdx.x < 2 * K) {
    long long s = 0;
#pragma unroll
    for (int q = 0; q < kTW; ++q) s += sh[threadIdx.x * kTW + q];
    const int word = word0 + threadIdx.x;
    if (x.world > 1 && ((all_mask >> (threadIdx.x >> 1)) & 1)) {
      for (int r = 0; r < x.world; ++r) red_sys_u64(x_acc(x, r, par) + word, s);
    } else {
      red_add_u64(local + word, s);
    }
  }
}

// red_cta_hilo over the update warps only (warps kUW..): named barrier 1,
// so the sums leave while warp 0 still runs the scalar logic
template <int NT, int K>
__device__ __forceinline__ void red_upd_hilo(HiLo (&v)[K], int word0, int all_mask,
                                             const XArgs& x, int par, long long* local,
                                             long long* sh) {
  constexpr int kTW = NT / 32;
  constexpr int kUT = NT - 32 * kUW;
  static_assert(K <= 8, "16 words per lane");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long w[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w[2 * k] = k < K ? v[k].hi : 0;
    w[2 * k + 1] = k < K ? v[k].lo : 0;
  }
  const long long ws = bfly16(w, lane);
  if ((lane & 1) == 0) sh[bfly16_word(lane) * kTW + warp] = ws;
  asm volatile("bar.sync 1, %0;" ::"n"(kUT) : "memory");
  const int t = threadIdx.x - 32 * kUW;
  if (t < 2 * K) {
    long long s = 0;
#pragma unroll
    for (int w2 = kUW; w2 < kTW; ++w2) s += sh[t * kTW + w2];
    const int word = word0 + t;
    if (x.world > 1 && ((all_mask >> (t >> 1)) & 1)) {
      for (int r = 0; r < x.world; ++r) red_sys_u64(x_acc(x, r, par) + word, s);
    } else {
      red_add_u64(local + word, s);
    }
  }
}

// the fixed-point row / column sums of the sweep (PassArgs::fx): fp32 one
// word at 2^46, fp64 a hi / lo pair (second half of the array)
template <class T>
__device__ __forceinline__ T fx_take(long long* fxa, int64_t i, int64_t len) {
  const long long hi = __ldcg(fxa + i);
  fxa[i] = 0;
  if (sizeof(T) == 4) return static_cast<T>(static_cast<double>(hi) * kFxInv);
  const long long lo = __ldcg(fxa + len + i);
  fxa[len + i] = 0;
  return static_cast<T>(static_cast<double>(hi) * kFxInv + static_cast<double>(lo) * kFxLoInv);
}

// One iteration's tail on NT-thread CTAs (the whole grid): the body of
// tail_kernel, and of the small-problem solver's loop.  Returns whether the
// solve stops (the decision every CTA holds identically).
template <class T, int NT>
__device__ __forceinline__ bool tail_body(const TailArgs<T>& t, unsigned* bar) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  constexpr int BW = static_cast<int>(sizeof(Book<T>) / 8);
  constexpr int UT = NT - 32 * kUW;      // update threads per CTA
  Book<T>* bk = t.book;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int par = t.tpar & 1;
  const XArgs& X = t.x;
  const bool multi = X.world > 1;  // row shards: counters / sums on every rank
  unsigned* ctr = bar + (par ? kCtr1 : kCtr0);
  // this iteration's accumulators and the other parity's (the previous
  // iteration's pending update sums, the next iteration's sweep / merge sums)
  long long* xa = multi ? x_acc(X, X.rank, par) : t.xacc + par * kXaWords;
  long long* xn = multi ? x_acc(X, X.rank, par ^ 1) : t.xacc + (par ^ 1) * kXaWords;
  // a stopped loop (graph batches run on past the stop): nothing to do, and
  // nothing may be reset -- the last iteration's pending update sums (P)
  // are still to be read by the finalize kernel
  if (*reinterpret_cast<volatile int*>(&bk->stop)) return true;
  // CTA 0 prepares what others (of every rank) only touch after barrier 1
  // or in the next launch: the next tail's counters and sweep / merge sums
  // (A of the other parity), this iteration's update and report sums (P, R)
  if (blockIdx.x == 0) {
    if (tid == 0) bar[par ? kCtr0 : kCtr1] = 0u;
    if (multi && tid < 4) *x_ctr(X, X.rank, par ^ 1, tid) = 0u;
    if (tid < kXaP) xn[tid] = 0;
    else if (tid < kXaWords) xa[tid] = 0;
  }
  const int64_t it_stamp = t.stamps ? *reinterpret_cast<volatile int64_t*>(&bk->iter) : 0;
  TAIL_STAMP(2);
  if (multi) {
    // row shards: this rank's sweep left fixed-point column partials in vfx
    // and its scalars in xloc -- add both into every rank's sums (integer
    // atomics over NVLink: exact, so the totals do not depend on the rank
    // count or order), then a cross-rank barrier
    const int64_t n_ = t.n;
    const int vw = X.vwords;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * NT + tid; j < n_;
         j += static_cast<int64_t>(gridDim.x) * NT) {
      for (int w = 0; w < vw; ++w) {
        const long long q = __ldcg(t.vfx + w * n_ + j);
        t.vfx[w * n_ + j] = 0;
        if (q != 0)
          for (int r = 0; r < X.world; ++r) red_sys_u64(x_vsum(X, r, par, n_) + w * n_ + j, q);
      }
    }
    if (blockIdx.x == 0 && tid < 2 * kXaDx + 2) {  // cost, prev, dual, dx (hi / lo)
      long long* src = t.xloc + par * kXaWords + tid;
      const long long q = __ldcg(src);
      *src = 0;
      for (int r = 0; r < X.world; ++r) red_sys_u64(x_acc(X, r, par) + tid, q);
    } else if (blockIdx.x == 0 && (tid == 32 || tid == 33)) {  // max |t|, non-finite count
      const int word = tid == 32 ? kXaMax : kXaBad;
      long long* src = t.xloc + par * kXaWords + word;
      const long long q = __ldcg(src);
      *src = 0;
      for (int r = 0; r < X.world; ++r) {
        if (tid == 32)
          red_sys_max_u64(x_acc(X, r, par) + word, q);
        else
          red_sys_u64(x_acc(X, r, par) + word, q);
      }
    }
    xrank_barrier(X, par, 0, static_cast<unsigned>(X.world) * gridDim.x, nullptr, 0);
  }
  __shared__ __align__(16) T red[NT * R];  // strip merge partition sums [P][CV][R]
  __shared__ Book<T> sbk;
  __shared__ long long shL[2 * 8 * 8];
  __shared__ long long shP[2 * 8 * 8];  // update sums (named-barrier reduction)
  __shared__ double s_tot[24];
  __shared__ DecideIn<T> s_din;  // tail_decide's inputs (thread 0 only)
  const int64_t m = t.m, n = t.n;
  const bool fg = t.fused_gate != 0;
  // the Book as this launch found it (CTA 0 of the previous tail or the host
  // wrote it; nobody writes it before barrier 1)
  if (tid < BW)
    reinterpret_cast<unsigned long long*>(&sbk)[tid] =
        __ldcg(reinterpret_cast<const unsigned long long*>(bk) + tid);
  const bool fp = bk->record_trace != 0;  // configuration: constant over the solve
  // tail_decide's launch constants (thread 0 runs the decision)
  if (fg && tid == 0) decide_consts<T>(&s_din, t);

  // this CTA's balanced range of [0, m + n): the update, and the merge in
  // fixed-point mode; update thread ut takes e0 + ut, e0 + ut + UT, ...
  const int64_t E = m + n;
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * E / G;
  const int64_t e1 = static_cast<int64_t>(blockIdx.x + 1) * E / G;
  const int ut = tid - 32 * kUW;
  const int64_t ef = e0 + ut;
  const bool has_first = ut >= 0 && ef < e1;
  // first element: its update inputs are independent of the merge -- load
  // them now (a / b, p / q, old phi / varphi, old r / s)
  T f_ab = T(0), f_pq = T(0), f_old = T(0), f_rso = T(0), f_rs = T(0);
  if (has_first) {
    if (ef < m) {
      f_ab = ld_keep(t.a + ef);
      f_pq = ld_keep(t.p + ef);
      f_old = ld_keep(t.phi + ef);
      if (fp) f_rso = ld_keep(t.r_old + ef);
    } else {
      const int64_t j = ef - m;
      f_ab = ld_keep(t.b + j);
      f_pq = ld_keep(t.q + j);
      f_old = ld_keep(t.varphi + j);
      if (fp) f_rso = ld_keep(t.s_old + j);
    }
  }

  // ---- A: merge: r = u - p, s = v - q and their exact sums ------------------
  // {sum r, |r|^2, |s|^2, sum p a, sum p r, sum q b, sum q s}
  HiLo hm[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) hm[k] = HiLo{0, 0};
  auto row_terms = [&](int64_t i, T ui, T pi, T ai) -> T {
    const T r = ui - pi;
    st_keep(t.r_new + i, r, 2);
    hilo_add(hm[0], static_cast<double>(r));
    hilo_add(hm[1], static_cast<double>(r * r));
    hilo_add(hm[3], static_cast<double>(pi) * static_cast<double>(ai));
    hilo_add(hm[4], static_cast<double>(pi) * static_cast<double>(r));
    return r;
  };
  auto col_terms = [&](int64_t j, T vj, T qj, T bj) -> T {
    const T sv = vj - qj;
    st_keep(t.s_new + j, sv, 2);
    hilo_add(hm[2], static_cast<double>(sv * sv));
    hilo_add(hm[5], static_cast<double>(qj) * static_cast<double>(bj));
    hilo_add(hm[6], static_cast<double>(qj) * static_cast<double>(sv));
    return sv;
  };
  if (t.fx) {
    // complete after the sweep: one read (and reset) per index, by the
    // update thread that owns it
    if (ut >= 0) {
      for (int64_t e = ef; e < e1; e += UT) {
        const bool first = e == ef;
        if (e < m) {
          const T pi = first ? f_pq : ld_keep(t.p + e);
          const T ai = first ? f_ab : ld_keep(t.a + e);
          const T r = row_terms(e, fx_take<T>(t.ufx, e, t.ld), pi, ai);
          if (first) f_rs = r;
        } else {
          const int64_t jj = e - m;
          const T qj = first ? f_pq : ld_keep(t.q + jj);
          const T bj = first ? f_ab : ld_keep(t.b + jj);
          const T sv = col_terms(
              jj, fx_take<T>(multi ? x_vsum(X, X.rank, par, n) : t.vfx, jj, n), qj, bj);
          if (first) f_rs = sv;
        }
      }
    }
  } else {
    // strips (a warm start): (m + n) merged sums as RV-wide vectors (16-B
    // loads), u vectors [0, nvu), v vectors [nvu, nvu + nvv); CTA b owns the
    // balanced range [b*NV/G, (b+1)*NV/G); thread t of a chunk of CV vectors
    // handles vector t % CV over the strip rows g = t / CV (mod P), 8 loads in
    // flight; the P partition sums are combined in a fixed order in shared
    // memory, then the chunk's owner thread forms r / s per element
    const int64_t nvu = (m + R - 1) / R, nvv = (n + R - 1) / R, NV = nvu + nvv;
    const bool vvec = (n % R) == 0;  // v strip rows 16-B aligned
    const int64_t v0 = static_cast<int64_t>(blockIdx.x) * NV / G;
    const int64_t v1 = static_cast<int64_t>(blockIdx.x + 1) * NV / G;
    const int64_t cnt = v1 - v0;
    int P = cnt > 0 ? static_cast<int>(NT / cnt) : 8;
    P = P < 1 ? 1 : (P > 8 ? 8 : P);
    const int CV = NT / P;
    T* redv = red;
    for (int64_t c0 = v0; c0 < v1; c0 += CV) {
      const int64_t vec = c0 + tid % CV;
      const int part = tid / CV;
      T acc[R];
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] = T(0);
      if (part < P && vec < v1) {
        const bool isu = vec < nvu;
        const int64_t rows = isu ? t.grid_cols : t.grid_rows64;
        const int64_t stride = isu ? t.ld : n;
        const T* base = isu ? t.ustrip + vec * R : t.vstrip + (vec - nvu) * R;
        if (isu || vvec) {
          const V* bv = reinterpret_cast<const V*>(base);
          const int64_t sv = stride / R;
          int64_t g = part;
          for (; g + 7 * P < rows; g += 8 * P) {
            V x8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) x8[q] = bv[(g + q * P) * sv];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              T e[R];
              unpack(x8[q], e);
#pragma unroll
              for (int k = 0; k < R; ++k) acc[k] += e[k];
            }
          }
          for (; g < rows; g += P) {
            T e[R];
            unpack(bv[g * sv], e);
#pragma unroll
            for (int k = 0; k < R; ++k) acc[k] += e[k];
          }
        } else {  // v strips of a row length that is not a multiple of R
          const int64_t j0 = (vec - nvu) * R;
          for (int64_t g = part; g < rows; g += P)
#pragma unroll
            for (int k = 0; k < R; ++k)
              if (j0 + k < n) acc[k] += base[g * stride + k];
        }
      }
      if (c0 == v0) TAIL_STAMP(7);
      __syncthreads();
      if (part < P)
#pragma unroll
        for (int k = 0; k < R; ++k) redv[(part * CV + tid % CV) * R + k] = acc[k];
      __syncthreads();
      if (tid < CV && vec < v1) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          T tot = T(0);
          for (int q = 0; q < P; ++q) tot += redv[(q * CV + tid) * R + k];
          if (vec < nvu) {
            const int64_t i = vec * R + k;
            if (i < m) row_terms(i, tot, ld_keep(t.p + i), ld_keep(t.a + i));
          } else {
            const int64_t j = (vec - nvu) * R + k;
            if (j < n) col_terms(j, tot, ld_keep(t.q + j), ld_keep(t.b + j));
          }
        }
      }
    }
  }
  TAIL_STAMP(8);
  red_cta_hilo_x<NT, 7>(hm, 2 * kXaSumR, 0x1B, X, par, xa, shL);
  TAIL_STAMP(3);
  // ---- barrier 1: every CTA reads the exact totals -------------------------
  if (multi)
    xrank_barrier(X, par, 1, static_cast<unsigned>(X.world) * G, t.stamps, it_stamp);
  else
    count_barrier(ctr, static_cast<unsigned>(G), t.stamps, it_stamp);
  // s_tot: [0, 11) the A sums, [11] max|t|, [12] non-finite count,
  // [13, 21) the previous iteration's P sums
  if (tid < 11) {
    s_tot[tid] = hilo_value(__ldcg(xa + 2 * tid), __ldcg(xa + 2 * tid + 1));
  } else if (tid == 11) {
    s_tot[11] = __longlong_as_double(__ldcg(xa + kXaMax));
  } else if (tid == 12) {
    s_tot[12] = static_cast<double>(__ldcg(xa + kXaBad));
  } else if (tid >= 32 && tid < 40 && fg) {
    const int k = tid - 32;
    s_tot[13 + k] = hilo_value(__ldcg(xn + kXaP + 2 * k), __ldcg(xn + kXaP + 2 * k + 1));
  }
  TAIL_STAMP(11);
  __syncthreads();
  // the pass totals in T, as the per-CTA sums of the sweep are
  const T tot8[8] = {static_cast<T>(s_tot[kXaCost]), static_cast<T>(s_tot[kXaPrev]),
                     static_cast<T>(s_tot[kXaDual]), static_cast<T>(s_tot[kXaDx]),
                     static_cast<T>(s_tot[11]),      static_cast<T>(s_tot[kXaSumR]),
                     static_cast<T>(s_tot[kXaR2]),   static_cast<T>(s_tot[kXaS2])};
  // coef exactly as merge_scalars forms it (solver.hpp:273-277), from the
  // Book before this iteration's scalar logic touches it
  const T beta_all = tot8[5] / static_cast<T>(t.m_global + t.n_global);
  const T coef = T(2) * beta_all - sbk.alpha;
  const bool pass_bad = s_tot[12] > 0.0;
  // the previous iteration's commit record, before warp 0 overwrites it
  CommitRec crec{};
  if (tid == 32) crec = commit_snap(sbk);
  __syncthreads();
  // warp 0: this iteration's decision (gate.cuh tail_decide); warp 1: the
  // previous iteration's commit and exact dual / fixed-point patch; warps
  // 2..: the update (solver.hpp:279-289) -- concurrently
  if (warp == 0) {
    if (lane == 0) {
      if (fg) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s_din.tot[q] = tot8[q];
        s_din.totbad = pass_bad ? 1 : 0;
        s_din.sum_pa = s_tot[kXaPA];
        s_din.sum_pr = s_tot[kXaPR];
        s_din.sum_qb = s_tot[kXaQB];
        s_din.sum_qs = s_tot[kXaQS];
        tail_decide<T>(&sbk, &s_din);
        sbk.pend_buf = par;
        TAIL_STAMP(15);
      } else {
        merge_scalars<T>(&sbk, t, tot8, pass_bad ? 1 : 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && fg && crec.valid) {
      tail_commit<T>(&sbk, t, crec, blockIdx.x == 0);
      const double d8[8] = {s_tot[13], s_tot[14], s_tot[15], s_tot[16],
                            s_tot[17], s_tot[18], s_tot[19], s_tot[20]};
      patch_pending<T>(&sbk, t, d8, blockIdx.x == 0);
    }
  }
  // ---- B: phi / varphi / a / b + exact dual-value and fixed-point sums ------
  HiLo hp[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) hp[k] = HiLo{0, 0};
  if (warp >= kUW && !pass_bad) {
    const T inv_n = T(1) / static_cast<T>(t.n_global);
    const T inv_m = T(1) / static_cast<T>(t.m_global);
    const double drho = static_cast<double>(t.rho);
    for (int64_t e = ef; e < e1; e += UT) {
      const bool first = e == ef && t.fx;
      if (e < m) {
        const T r = first ? f_rs : ld_keep_cg(t.r_new + e);
        const T ph_old = e == ef ? f_old : ld_keep(t.phi + e);
        const T ai = e == ef ? f_ab : ld_keep(t.a + e);
        const T pi = e == ef ? f_pq : ld_keep(t.p + e);
        const T ph = (ai - T(2) * r + coef) * inv_n;  // solver.hpp:280-282
        st_keep(t.phi + e, ph, 2);
        st_keep(t.a + e, ai - r, 2);  // solver.hpp:287
        hilo_add(hp[0], static_cast<double>(pi) * static_cast<double>(ph) / drho);
        if (fp) {
          const T ro = e == ef ? f_rso : ld_keep(t.r_old + e);
          const double d = static_cast<double>(ph) - static_cast<double>(ph_old);
          hilo_add(hp[1], d * d);
          hilo_add(hp[2], d);
          hilo_add(hp[3], d * (static_cast<double>(r) - static_cast<double>(ro)));
        }
      } else {
        const int64_t j = e - m;
        const T sv = first ? f_rs : ld_keep_cg(t.s_new + j);
        const T vp_old = e == ef ? f_old : ld_keep(t.varphi + j);
        const T bj = e == ef ? f_ab : ld_keep(t.b + j);
        const T qj = e == ef ? f_pq : ld_keep(t.q + j);
        const T vp = (bj - T(2) * sv + coef) * inv_m;  // solver.hpp:283-285
        st_keep(t.varphi + j, vp, 2);
        st_keep(t.b + j, bj - sv, 2);  // solver.hpp:288
        hilo_add(hp[4], static_cast<double>(qj) * static_cast<double>(vp) / drho);
        if (fp) {
          const T so = e == ef ? f_rso : ld_keep(t.s_old + j);
          const double d = static_cast<double>(vp) - static_cast<double>(vp_old);
          hilo_add(hp[5], d * d);
          hilo_add(hp[6], d);
          hilo_add(hp[7], d * (static_cast<double>(sv) - static_cast<double>(so)));
        }
      }
    }
  }
  if (t.stamps && tid == 32 * kUW) timeline_point(t.stamps, it_stamp, 13, global_ns());
  if (warp >= kUW && !pass_bad) red_upd_hilo<NT, 8>(hp, kXaP, 0x0F, X, par, xa, shP);
  if (t.stamps && tid == 32 * kUW) timeline_point(t.stamps, it_stamp, 14, global_ns());
  __syncthreads();
  TAIL_STAMP(12);
  book_store_cta0(bk, &sbk);
  TAIL_STAMP(4);
  __syncthreads();
  TAIL_STAMP(5);
  if (sbk.failed) return true;  // non-finite pass
  if (fg && (!sbk.confirm || sbk.stop == 1)) {
    TAIL_STAMP(6);
    return sbk.stop != 0;
  }
  // ---- barrier 2 (only when needed): exact dual value / exact gate ----------
  if (multi)
    xrank_barrier(X, par, 2, static_cast<unsigned>(X.world) * G, nullptr, 0);
  else
    count_barrier(ctr, 2u * static_cast<unsigned>(G), nullptr, 0);
  if (tid < 8) s_tot[13 + tid] = hilo_value(__ldcg(xa + kXaP + 2 * tid), __ldcg(xa + kXaP + 2 * tid + 1));
  __syncthreads();
  if (tid == 0) {
    const double d8[8] = {s_tot[13], s_tot[14], s_tot[15], s_tot[16],
                          s_tot[17], s_tot[18], s_tot[19], s_tot[20]};
    if (fg) {
      // this iteration's commit now (its record is consumed: the next tail
      // must not apply it again), then its exact dual value and the
      // reference's gap test before the report
      const CommitRec c = commit_snap(sbk);
      tail_commit<T>(&sbk, t, c, blockIdx.x == 0);
      sbk.cm_valid = 0;
      patch_pending<T>(&sbk, t, d8, blockIdx.x == 0);
      gate_recheck<T>(&sbk);
    } else {
      gate_logic<T>(&sbk, t, d8[0] + d8[4], d8[1], d8[2], d8[5], d8[6], d8[3] + d8[7],
                    blockIdx.x == 0);
    }
  }
  book_store_cta0(bk, &sbk);
  __syncthreads();
  if (!sbk.confirm || sbk.stop == 1) return sbk.stop != 0;

  // ---- C: exact confirm report (only when the gate fired) ------------------
  {
    const bool folded = sbk.folded != 0;
    const double drho = static_cast<double>(t.rho);
    const int64_t ngx = (m + int64_t(NT) * R - 1) / (int64_t(NT) * R);
    const int64_t ncs = imin64(n, (2 * static_cast<int64_t>(G) + ngx - 1) / ngx);
    HiLo hr[2] = {HiLo{0, 0}, HiLo{0, 0}};
    for (int64_t unit = blockIdx.x; unit < ngx * ncs; unit += G) {
      const int64_t rx = unit % ngx, cs = unit / ngx;
      const int64_t row0 = (rx * NT + tid) * R;
      if (row0 >= m) continue;
      const int nvalid = static_cast<int>(imin64(R, m - row0));
      double mu[R];
#pragma unroll
      for (int k = 0; k < R; ++k)
        mu[k] = k < nvalid ? static_cast<double>(__ldcg(t.phi + row0 + k)) / drho : 0.0;
      for (int64_t j = cs; j < n; j += ncs) {
        const double nu_j = static_cast<double>(__ldcg(t.varphi + j)) / drho;
        T xv[R], cv[R];
        unpack(__ldcs(reinterpret_cast<const V*>(t.report_x + j * t.ld + row0)), xv);
        unpack(__ldcs(reinterpret_cast<const V*>(t.report_c + j * t.ld + row0)), cv);
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (k < nvalid)
            report_elem_exact<T>(xv[k], cv[k], mu[k], nu_j, t.rho, folded, hr);
      }
    }
    red_cta_hilo_x<NT, 2>(hr, kXaR, 0x3, X, par, xa, shL);
  }
  if (multi)
    xrank_barrier(X, par, 3, static_cast<unsigned>(X.world) * G, nullptr, 0);
  else
    count_barrier(ctr, 3u * static_cast<unsigned>(G), nullptr, 0);
  if (tid < 2) s_tot[tid] = hilo_value(__ldcg(xa + kXaR + 2 * tid), __ldcg(xa + kXaR + 2 * tid + 1));
  __syncthreads();
  if (tid == 0) report_decide<T>(&sbk, s_tot[0], s_tot[1], 0);
  book_store_cta0(bk, &sbk);
  return sbk.stop != 0;
}

template <class T>
__global__ void __launch_bounds__(kTT) tail_kernel(const TailArgs<T> t, unsigned* bar) {
  // the next sweep (a programmatic dependent) may be scheduled now; it waits
  // in griddepcontrol.wait for this grid's completion
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (t.pdl: after the sweep)
  tail_body<T, kTT>(t, bar);
}

// ---------------------------------------------------------------------------
// KC: the same tail as ONE thread-block cluster (16 -- or 8 -- CTAs of
// kCT threads in one GPC), for a single GPU in fixed-point mode when m + n
// fits the updating CTAs' threads (kCK elements each: 26 880 at 16 CTAs).
// The grid tail's global round trips per reduction (arrival atomics + spin on
// an L2 counter, then a load of the totals) become hardware cluster barriers
// and distributed-shared-memory reads; the 16 CTAs leave 132 SMs to the next
// sweep, whose CTAs (programmatic dependents) become resident and prime their
// rings while the tail runs.  The exact integer sums make the totals
// independent of the partition, so KC and the grid tail give bit-identical
// iterations (tests/test_tail_gpu.py).
//   prologue  Book, the sweep's exact totals (complete: kernel boundary) and
//             the previous iteration's update sums; each update thread of
//             CTAs 1.. loads its <= kCK elements' inputs at once; then the
//             stop flag
//   A  merge  (CTAs 1..) r = u - p, s = v - q from the fixed-point sums; CTA
//             partials of the 7 merge sums -> cluster barrier 1 -> every CTA
//             adds the C partials over DSMEM (same totals everywhere)
//   B  CTA 0, thread 0: the decision, pushed to every CTA's shared memory;
//      thread 32: the previous iteration's commit and patch.  CTAs 1..,
//      warps 2..: the update + its 8 exact sums, added into CTA 0's shared
//      memory (DSMEM atomics) -> cluster barrier 2 -> CTA 0 stores the sums
//      and the Book
//   C  (only when the gate fired) exact dual value, recheck and the exact
//      report over the cluster, reduced the same way
// ---------------------------------------------------------------------------
constexpr int kCT = 512;                 // threads per cluster CTA (256 for small m + n)
constexpr int kCK = 4;                   // elements per update thread (at most)

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_ctas() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// every thread of every CTA of the cluster; release / acquire at cluster scope
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of this CTA's shared variable `p` in CTA `r` of the cluster
__device__ __forceinline__ uint32_t dsmem(const void* p, unsigned r) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(a), "r"(r));
  return out;
}
__device__ __forceinline__ long long ld_dsmem(uint32_t a) {
  long long v;
  asm volatile("ld.relaxed.cluster.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_dsmem_s32(uint32_t a, int v) {
  asm volatile("st.relaxed.cluster.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_dsmem(uint32_t a, long long v) {
  asm volatile("red.relaxed.cluster.shared::cluster.add.u64 [%0], %1;" ::"r"(a), "l"(v)
               : "memory");
}

// per-CTA sums of K <= 8 HiLo values over the threads [32 * W0, NT): a warp
// reduce-scatter (bfly16), then thread 32 * W0 + w adds word w over the
// warps.  sync(): the barrier over exactly those threads.
template <int NT, int K, int W0, class Sync>
__device__ __forceinline__ long long cta_sum_hilo(HiLo (&v)[K], long long* sh, Sync sync) {
  constexpr int kW = NT / 32;
  static_assert(K <= 8, "16 words per lane");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long w[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w[2 * k] = k < K ? v[k].hi : 0;
    w[2 * k + 1] = k < K ? v[k].lo : 0;
  }
  const long long ws = bfly16(w, lane);
  if ((lane & 1) == 0) sh[bfly16_word(lane) * kW + warp] = ws;
  sync();
  const int t = threadIdx.x - 32 * W0;
  long long s = 0;
  if (t >= 0 && t < 2 * K)
#pragma unroll
    for (int q = W0; q < kW; ++q) s += sh[t * kW + q];
  return s;
}

template <class T, int NT>
__global__ void __launch_bounds__(NT, 1) ctail_kernel(const TailArgs<T> t) {
  constexpr int kCT = NT;
  constexpr int kCUT = NT - 32 * kUW;  // update threads per CTA
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int BW = static_cast<int>(sizeof(Book<T>) / 8);
  constexpr int kW = kCT / 32;
  Book<T>* bk = t.book;
  const int tid = threadIdx.x, warp = tid >> 5;
  const unsigned C = cluster_ctas(), cr = cluster_rank();
  const bool lead = cr == 0;  // CTA 0 decides and keeps the Book; CTAs 1.. update
  const int par = t.tpar & 1;
  long long* xa = t.xacc + par * kXaWords;
  long long* xn = t.xacc + (par ^ 1) * kXaWords;
  __shared__ Book<T> sbk;
  __shared__ DecideIn<T> s_din;
  __shared__ double s_tot[24];
  __shared__ long long sh[2 * 8 * kW];
  __shared__ long long s_part[16];  // this CTA's 7 merge sums (hi / lo)
  __shared__ long long s_word[16];  // their cluster totals
  __shared__ long long s_P[16];     // CTA 0: the cluster's 8 update sums
  __shared__ long long s_R[4];      // CTA 0: the 2 report sums
  __shared__ int s_flags;           // CTA 0's decision: failed | confirm << 1 | stop << 2
  __shared__ CommitIn s_cin;        // CTA 0: commit_patch's inputs
  const int64_t it_stamp = t.stamps ? *reinterpret_cast<volatile int64_t*>(&bk->iter) : 0;
  TAIL_STAMP(2);
  if (tid < BW) {
    const unsigned long long w = __ldcg(reinterpret_cast<const unsigned long long*>(bk) + tid);
    reinterpret_cast<unsigned long long*>(&sbk)[tid] = w;
  }
  if (lead) {
    if (tid >= 32 && tid < 48) s_P[tid - 32] = 0;
    if (tid >= 64 && tid < 68) s_R[tid - 64] = 0;
  }
  // the sweep's totals (complete: kernel boundary) and the previous
  // iteration's update sums (P of the other parity)
  if (tid < 4) {
    s_tot[tid] = hilo_value(__ldcg(xa + 2 * tid), __ldcg(xa + 2 * tid + 1));
  } else if (tid == 4) {
    s_tot[11] = __longlong_as_double(__ldcg(xa + kXaMax));
  } else if (tid == 5) {
    s_tot[12] = static_cast<double>(__ldcg(xa + kXaBad));
  } else if (tid == 6 && lead) {
    decide_consts<T>(&s_din, t);
  } else if (tid >= 32 && tid < 40 && lead) {
    const int k = tid - 32;
    s_tot[13 + k] = hilo_value(__ldcg(xn + kXaP + 2 * k), __ldcg(xn + kXaP + 2 * k + 1));
  }
  const bool fp = bk->record_trace != 0;
  const int64_t m = t.m, n = t.n, E = m + n;
  // CTAs 1..C-1 share [0, m + n); update thread ut takes e0 + ut + k * kCUT
  const int64_t e0 = lead ? 0 : static_cast<int64_t>(cr - 1) * E / (C - 1);
  const int64_t e1 = lead ? 0 : static_cast<int64_t>(cr) * E / (C - 1);
  const int ut = tid - 32 * kUW;
  // element e is row e (e < m) or column e - m: the same code for both, on
  // selected pointers (one compact body -- the tail's code is fetched cold
  // every iteration, so its size is latency)
  T f_ab[kCK], f_pq[kCK], f_old[kCK], f_rso[kCK], f_rs[kCK];
  long long fxh[kCK], fxl[kCK];
#pragma unroll
  for (int k = 0; k < kCK; ++k) {
    f_ab[k] = f_pq[k] = f_old[k] = f_rso[k] = f_rs[k] = T(0);
    fxh[k] = fxl[k] = 0;
    const int64_t e = e0 + ut + static_cast<int64_t>(k) * kCUT;
    if (ut < 0 || e >= e1) continue;
    const bool row = e < m;
    const int64_t i = row ? e : e - m;
    const long long* fxa = row ? t.ufx : t.vfx;
    fxh[k] = __ldcg(fxa + i);
    if (sizeof(T) == 8) fxl[k] = __ldcg(fxa + (row ? t.ld : n) + i);
    f_ab[k] = ld_keep((row ? t.a : t.b) + i);
    f_pq[k] = ld_keep((row ? t.p : t.q) + i);
    f_old[k] = ld_keep((row ? t.phi : t.varphi) + i);
    f_rso[k] = ld_keep((row ? t.r_old : t.s_old) + i);  // (used when fp)
  }
  // a stopped loop: nothing to do and nothing may be written (every CTA reads
  // the same flag: the Book is only written after cluster barrier 2).  Read
  // after the loads above are in flight, so its latency overlaps theirs.
  if (*reinterpret_cast<volatile int*>(&bk->stop)) return;
  if (lead && tid < kXaP) xn[tid] = 0;  // the next sweep's accumulators
  TAIL_STAMP(8);
  // ---- A: merge (solver.hpp:269-272) and its exact sums ----------------------
  // {sum r, |r|^2, |s|^2, sum p a, sum p r, sum q b, sum q s}
  // (the updating CTAs' path first: the code of a kernel is fetched on
  // demand, and the hot path placed first in the text measured ~3 us faster
  // per tail than behind CTA 0's block)
  if (!lead) {
    HiLo hm[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) hm[k] = HiLo{0, 0};
#pragma unroll
    for (int k = 0; k < kCK; ++k) {
      const int64_t e = e0 + ut + static_cast<int64_t>(k) * kCUT;
      if (ut < 0 || e >= e1) continue;
      const bool row = e < m;
      const int64_t i = row ? e : e - m;
      long long* fxa = row ? t.ufx : t.vfx;
      const double fv = sizeof(T) == 4 ? static_cast<double>(fxh[k]) * kFxInv
                                       : static_cast<double>(fxh[k]) * kFxInv +
                                             static_cast<double>(fxl[k]) * kFxLoInv;
      fxa[i] = 0;
      if (sizeof(T) == 8) fxa[(row ? t.ld : n) + i] = 0;
      const T rs = static_cast<T>(fv) - f_pq[k];  // r = u - p, s = v - q
      st_keep((row ? t.r_new : t.s_new) + i, rs, 2);
      // rows: sum r, |r|^2, sum p a, sum p r; columns: |s|^2, sum q b, sum q s
      const HiLo h0 = to_hilo(static_cast<double>(rs));
      const HiLo h1 = to_hilo(static_cast<double>(rs * rs));
      const HiLo h2 = to_hilo(static_cast<double>(f_pq[k]) * static_cast<double>(f_ab[k]));
      const HiLo h3 = to_hilo(static_cast<double>(f_pq[k]) * static_cast<double>(rs));
      if (row) {
        hm[0].hi += h0.hi; hm[0].lo += h0.lo;
        hm[1].hi += h1.hi; hm[1].lo += h1.lo;
        hm[3].hi += h2.hi; hm[3].lo += h2.lo;
        hm[4].hi += h3.hi; hm[4].lo += h3.lo;
      } else {
        hm[2].hi += h1.hi; hm[2].lo += h1.lo;
        hm[5].hi += h2.hi; hm[5].lo += h2.lo;
        hm[6].hi += h3.hi; hm[6].lo += h3.lo;
      }
      f_rs[k] = rs;
    }
    const long long s = cta_sum_hilo<kCT, 7, 0>(hm, sh, [] { __syncthreads(); });
    if (tid < 14) s_part[tid] = s;
    TAIL_STAMP(3);
    cluster_sync_all();  // (1) every CTA's merge partials are in its shared memory
  } else {
    // CTA 0 has no elements (it runs the scalar logic after the barrier)
    if (tid < 16) s_part[tid] = 0;
    TAIL_STAMP(3);
    cluster_sync_all();
  }
  TAIL_STAMP(10);
  if (tid < 14) {  // word tid over the C CTAs: 16 loads in flight (C = 8 or 16)
    long long v[16];
#pragma unroll
    for (unsigned c = 0; c < 16; ++c) v[c] = ld_dsmem(dsmem(&s_part[tid], c & (C - 1)));
    long long sum = 0;
#pragma unroll
    for (unsigned c = 0; c < 16; ++c) sum += c < C ? v[c] : 0;
    s_word[tid] = sum;
  }
  __syncthreads();
  if (tid < 7) s_tot[kXaSumR + tid] = hilo_value(s_word[2 * tid], s_word[2 * tid + 1]);
  __syncthreads();
  TAIL_STAMP(11);
  const T tot8[8] = {static_cast<T>(s_tot[kXaCost]), static_cast<T>(s_tot[kXaPrev]),
                     static_cast<T>(s_tot[kXaDual]), static_cast<T>(s_tot[kXaDx]),
                     static_cast<T>(s_tot[11]),      static_cast<T>(s_tot[kXaSumR]),
                     static_cast<T>(s_tot[kXaR2]),   static_cast<T>(s_tot[kXaS2])};
  const bool pass_bad = s_tot[12] > 0.0;
  // the previous iteration's commit record, before the decision overwrites it
  CommitRec crec{};
  if (lead && tid == 32) crec = commit_snap(sbk);
  __syncthreads();
  // ---- B: CTA 0: decision (warp 0) | commit + patch (warp 1);
  //         CTAs 1..: the update (warps 2..) ------------------------------------
  if (!lead) {
    if (warp >= kUW) {
      // coef as merge_scalars forms it (solver.hpp:273-277)
      const T beta_all = tot8[5] / static_cast<T>(t.m_global + t.n_global);
      const T coef = T(2) * beta_all - sbk.alpha;
      HiLo hp[8];
  #pragma unroll
      for (int k = 0; k < 8; ++k) hp[k] = HiLo{0, 0};
      if (!pass_bad) {
        const T inv_n = T(1) / static_cast<T>(t.n_global);
        const T inv_m = T(1) / static_cast<T>(t.m_global);
        const double drho = static_cast<double>(t.rho);
#pragma unroll
        for (int k = 0; k < kCK; ++k) {
          const int64_t e = e0 + ut + static_cast<int64_t>(k) * kCUT;
          if (e >= e1) continue;
          const bool row = e < m;
          const int64_t i = row ? e : e - m;
          // phi = (a - 2 r + coef) / n, varphi = (b - 2 s + coef) / m
          // (solver.hpp:280-285); a -= r, b -= s (solver.hpp:287-288)
          const T ph = (f_ab[k] - T(2) * f_rs[k] + coef) * (row ? inv_n : inv_m);
          st_keep((row ? t.phi : t.varphi) + i, ph, 2);
          st_keep((row ? t.a : t.b) + i, f_ab[k] - f_rs[k], 2);
          const double d = static_cast<double>(ph) - static_cast<double>(f_old[k]);
          const HiLo g0 = to_hilo(static_cast<double>(f_pq[k]) * static_cast<double>(ph) / drho);
          const int o = row ? 0 : 4;
#pragma unroll
          for (int q = 0; q < 8; q += 4)
            if (o == q) {
              hp[q].hi += g0.hi;
              hp[q].lo += g0.lo;
            }
          if (fp) {
            const HiLo g1 = to_hilo(d * d), g2 = to_hilo(d);
            const HiLo g3 = to_hilo(d * (static_cast<double>(f_rs[k]) - static_cast<double>(f_rso[k])));
#pragma unroll
            for (int q = 0; q < 8; q += 4)
              if (o == q) {
                hp[q + 1].hi += g1.hi; hp[q + 1].lo += g1.lo;
                hp[q + 2].hi += g2.hi; hp[q + 2].lo += g2.lo;
                hp[q + 3].hi += g3.hi; hp[q + 3].lo += g3.lo;
              }
          }
        }
      }
      if (t.stamps && tid == 32 * kUW) timeline_point(t.stamps, it_stamp, 13, global_ns());
      const long long s = cta_sum_hilo<kCT, 8, kUW>(hp, sh, [] {
        asm volatile("bar.sync 1, %0;" ::"n"(kCUT) : "memory");
      });
      if (ut < 16 && s != 0) red_dsmem(dsmem(&s_P[ut], 0), s);
      if (t.stamps && tid == 32 * kUW) timeline_point(t.stamps, it_stamp, 14, global_ns());
    }
  } else {
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) s_din.tot[q] = tot8[q];
      s_din.totbad = pass_bad ? 1 : 0;
      s_din.sum_pa = s_tot[kXaPA];
      s_din.sum_pr = s_tot[kXaPR];
      s_din.sum_qb = s_tot[kXaQB];
      s_din.sum_qs = s_tot[kXaQS];
      tail_decide<T>(&sbk, &s_din);
      sbk.pend_buf = par;
      const int f = (sbk.failed ? 1 : 0) | (sbk.confirm ? 2 : 0) | (sbk.stop << 2);
      for (unsigned c = 0; c < C; ++c) st_dsmem_s32(dsmem(&s_flags, c), f);
      TAIL_STAMP(15);
    } else if (tid == 32 && crec.valid) {
      // the previous iteration's commit and exact dual / fixed-point patch
      // (it reads nothing the decision writes)
      s_cin.c = crec;
#pragma unroll
      for (int k = 0; k < 8; ++k) s_cin.d8[k] = s_tot[13 + k];
      s_cin.trace = t.trace;
      s_cin.n_global = t.n_global;
      s_cin.m_global = t.m_global;
      s_cin.write_trace = 1;
      commit_patch<T>(&sbk, &s_cin);
    }
  }
  cluster_sync_all();  // (2) the update sums are in CTA 0, the decision everywhere
  TAIL_STAMP(12);
  if (lead && tid < 16) xa[kXaP + tid] = s_P[tid];
  book_store_cta0(bk, &sbk);
  TAIL_STAMP(4);
  if ((s_flags & 1) || !(s_flags & 2) || (s_flags >> 2) == 1) {
    TAIL_STAMP(6);
    return;  // (no CTA reads another's shared memory after barrier 2)
  }
  // ---- C: the gate fired: exact dual value and the reference's gap test -----
  if (lead && tid == 0) {
    double d8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) d8[k] = hilo_value(s_P[2 * k], s_P[2 * k + 1]);
    const CommitRec c = commit_snap(sbk);
    tail_commit<T>(&sbk, t, c, true);
    sbk.cm_valid = 0;
    patch_pending<T>(&sbk, t, d8, true);
    gate_recheck<T>(&sbk);
    const int f = (sbk.confirm ? 2 : 0) | (sbk.stop << 2);
    for (unsigned cc = 0; cc < C; ++cc) st_dsmem_s32(dsmem(&s_flags, cc), f);
  }
  book_store_cta0(bk, &sbk);
  cluster_sync_all();  // (3) the recheck's flags are everywhere
  if (!(s_flags & 2) || (s_flags >> 2) == 1) return;
  // exact confirm report of (X_{k+1}, phi / rho, varphi / rho) over the cluster
  {
    using V = typename V16<T>::type;
    constexpr int R = 16 / sizeof(T);
    const bool folded = t.folded_after != 0;
    const double drho = static_cast<double>(t.rho);
    const int64_t ngx = (m + int64_t(kCT) * R - 1) / (int64_t(kCT) * R);
    const int64_t ncs = imin64(n, (2 * static_cast<int64_t>(C) + ngx - 1) / ngx);
    HiLo hr[2] = {HiLo{0, 0}, HiLo{0, 0}};
    for (int64_t unit = cr; unit < ngx * ncs; unit += C) {
      const int64_t rx = unit % ngx, cs = unit / ngx;
      const int64_t row0 = (rx * kCT + tid) * R;
      if (row0 >= m) continue;
      const int nvalid = static_cast<int>(imin64(R, m - row0));
      double mu[R];
#pragma unroll
      for (int k = 0; k < R; ++k)
        mu[k] = k < nvalid ? static_cast<double>(__ldcg(t.phi + row0 + k)) / drho : 0.0;
      for (int64_t j = cs; j < n; j += ncs) {
        const double nu_j = static_cast<double>(__ldcg(t.varphi + j)) / drho;
        T xv[R], cv[R];
        unpack(__ldcs(reinterpret_cast<const V*>(t.report_x + j * t.ld + row0)), xv);
        unpack(__ldcs(reinterpret_cast<const V*>(t.report_c + j * t.ld + row0)), cv);
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (k < nvalid) report_elem_exact<T>(xv[k], cv[k], mu[k], nu_j, t.rho, folded, hr);
      }
    }
    __syncthreads();  // sh is reused
    const long long s = cta_sum_hilo<kCT, 2, 0>(hr, sh, [] { __syncthreads(); });
    if (tid < 4 && s != 0) red_dsmem(dsmem(&s_R[tid], 0), s);
  }
  cluster_sync_all();  // (4) the report sums are in CTA 0
  if (!lead) return;
  if (tid == 0)
    report_decide<T>(&sbk, hilo_value(s_R[0], s_R[1]), hilo_value(s_R[2], s_R[3]), 0);
  book_store_cta0(bk, &sbk);
}

}  // namespace

// ---------------------------------------------------------------------------
// Row shards: the per-iteration exchange fused into the tail over NVLink
// peer memory (no NCCL in the iteration loop).
//
//   A  local merge: r (local rows), the local column partial of v -- written
//      straight into slot `rank` of EVERY peer's receive buffer (NVLink
//      stores) -- and the local scalar partials
//   -- reduce-barrier; its last CTA writes the 16 scalar payload doubles to
//      every peer, fences at system scope, raises its generation flag on
//      every peer (st.release.sys) and waits until all `world` flags of its
//      own buffer reach this iteration (ld.acquire.sys) --
//   B  v_j = sum over ranks r = 0..world-1 of slot r (a FIXED order: every
//      rank computes bit-identical column sums, independent of timing),
//      s = v - q (replicated), closed-form dual column terms
//   -- reduce-barrier: global scalars (payloads summed in rank order),
//      recursions, patch of the previous trace row, fused gate (a fire
//      pauses the loop for the collective confirm report, stop = 2) --
//   C  phi (local rows), varphi (all columns, replicated), a, b, pending
//      update partials (row part travels in the next payload)
//
// Receive buffers alternate with the iteration parity: a rank can run at
// most one exchange ahead of any peer (it cannot pass the next flag wait
// before that peer has consumed the previous buffer), so two suffice.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ char* xslot(const XArgs& x, int peer, int buf, int slot) {
  return x.peers[peer] + kXIterOff + buf * x.buf_bytes + slot * x.slot_bytes;
}

// Setup collectives (init sums, error agreement, confirm report): one CTA
// writes this rank's vector into slot `rank` of every peer, raises its
// setup flag there and reduces the world slots of its own buffer in rank
// order once every flag reached `gen`.  Parity buffers as for the iteration
// exchange.
template <class U>
__global__ void __launch_bounds__(1024) xallreduce_kernel(const U* in, U* out, int64_t count,
                                                          int op, char* const* peers, int world,
                                                          int rank, int64_t setup_off,
                                                          int64_t setup_bytes,
                                                          unsigned long long gen) {
  const int pb = static_cast<int>(gen & 1);
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    const U v = in[i];
    for (int r = 0; r < world; ++r)
      reinterpret_cast<U*>(peers[r] + setup_off + (pb * world + rank) * setup_bytes)[i] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int r = 0; r < world; ++r)
      st_release_sys_u64(reinterpret_cast<unsigned long long*>(peers[r] + kXSetupFlagOff) + rank,
                         gen);
    const unsigned long long* mine =
        reinterpret_cast<const unsigned long long*>(peers[rank] + kXSetupFlagOff);
    for (int r = 0; r < world; ++r)
      while (ld_acquire_sys_u64(mine + r) < gen) {
      }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    U acc = U(0);
    for (int r = 0; r < world; ++r) {
      const U v = *reinterpret_cast<volatile const U*>(
          reinterpret_cast<const U*>(peers[rank] + setup_off + (pb * world + r) * setup_bytes) + i);
      acc = (r == 0) ? v : (op == 0 ? acc + v : (v > acc ? v : acc));
    }
    out[i] = acc;
  }
}

template <class T>
__global__ void __launch_bounds__(kTT) tail_finalize_kernel(const TailArgs<T> t) {
  // end of a run: the last iteration's commit and exact dual / fixed-point patch
  Book<T>* bk = t.book;
  if (threadIdx.x != 0) return;
  if (!*reinterpret_cast<volatile int*>(&bk->cm_valid) &&
      !*reinterpret_cast<volatile int*>(&bk->pend_valid))
    return;
  Book<T> lb = *bk;
  if (lb.cm_valid) {
    const CommitRec c = commit_snap(lb);
    tail_commit<T>(&lb, t, c, true);
    lb.cm_valid = 0;
  }
  if (lb.pend_valid) {
    const long long* xp = t.xacc + lb.pend_buf * kXaWords + kXaP;
    double d8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) d8[k] = hilo_value(xp[2 * k], xp[2 * k + 1]);
    patch_pending<T>(&lb, t, d8);
  }
  *bk = lb;
}

template <class T>
int tail_grid(int device) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  // An SM runs CTAs of kernels with different shared-memory carveouts only
  // after reconfiguring, i.e. once it is empty: a spinning tail CTA on an
  // SM configured for little shared memory would keep K1 (66 KB per CTA)
  // off that SM for good -- with shards of one process sharing a device
  // that is a deadlock.  The tails ask for the maximum carveout, K1's.
  cudaFuncSetAttribute(tail_kernel<T>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tail_kernel<T>, kTT, 0);
  // one CTA per SM: the last CTA reduces half as many partial rows; measured
  // 35 vs 39 us per iteration at 1000^2 fp64, equal at 10k^2 (r1n)
  int want = 1;
  if (const char* e = std::getenv("DROTB_TAIL_CTAS")) want = std::atoi(e);  // tuning aid
  if (want < 1) want = 1;
  if (const char* e = std::getenv("DROTB_TAIL_GRID")) {  // test aid: absolute grid size
    const int g = std::atoi(e);
    if (g >= 1 && g <= sms * per) return g;
  }
  return sms * (per < want ? per : want);
}

// CTAs per cluster of the cluster tail on `device`: 16 (a non-portable
// size) when such a cluster of kCT-thread CTAs can be resident, else 8, else 0
template <class T>
int ctail_ctas(int device) {
  for (void* f : {reinterpret_cast<void*>(ctail_kernel<T, kCT>),
                  reinterpret_cast<void*>(ctail_kernel<T, kCT / 2>)}) {
    cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
  }
  static std::atomic<int> cache[64];  // per device: 0 unknown, else size + 1
  std::atomic<int>& slot = cache[device & 63];
  const int got = slot.load(std::memory_order_acquire);
  if (got > 0) return got - 1;
  int size = 0;
  for (const int c : {16, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(c));
    cfg.blockDim = dim3(kCT);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(c);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, ctail_kernel<T, kCT>, &cfg) == cudaSuccess &&
        nc > 0) {
      size = c;
      break;
    }
  }
  (void)cudaGetLastError();
  slot.store(size + 1, std::memory_order_release);
  return size;
}

template <class T>
cudaError_t launch_tail(const TailArgs<T>& t, T* cpart, double* dpart, unsigned* bar, int grid,
                        cudaStream_t st) {
  // one GPU, fixed-point sums, fused gate, m + n within the cluster's update
  // threads: the cluster tail (same results, shorter critical path)
  if (t.ctail > 0 && t.x.world <= 1 && !t.sharded && t.fx && t.fused_gate && !t.pdl) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int hw = ctail_ctas<T>(dev);
    const int c = hw < t.ctail ? hw : t.ctail;
    // half-size CTAs when every element still gets its own thread (cheaper
    // CTA barriers and reductions where the tail is latency-bound: 14.3 vs
    // 14.5 us per iteration at 1000^2 fp64; with more elements per thread
    // they lose, 61.9 vs 59.6 at 5000^2 fp32 -- same-box A/B)
    const int64_t need = t.m + t.n;
    const int nt = need <= static_cast<int64_t>(c - 1) * (kCT / 2 - 32 * kUW) ? kCT / 2 : kCT;
    if (c > 0 && need <= static_cast<int64_t>(c - 1) * (kCT - 32 * kUW) * kCK) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(c));
      cfg.blockDim = dim3(nt);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = static_cast<unsigned>(c);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      count_launch();
      return nt == kCT ? cudaLaunchKernelEx(&cfg, ctail_kernel<T, kCT>, t)
                       : cudaLaunchKernelEx(&cfg, ctail_kernel<T, kCT / 2>, t);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kTT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = t.pdl ? 2 : 1;  // t.pdl: a programmatic dependent of the sweep
  // test aid: several shards of ONE process on ONE device run their tails
  // concurrently; the driver does not overlap two cooperative grids, so the
  // in-process test launches ordinary grids small enough to be co-resident
  const char* nc = std::getenv("DROTB_TAIL_NONCOOP");
  if (nc && nc[0] == '1' && t.x.world > 1) cfg.numAttrs = 0;
  count_launch();
  (void)cpart;
  (void)dpart;
  return cudaLaunchKernelEx(&cfg, tail_kernel<T>, t, bar);
}

template <class U>
void launch_xallreduce(const U* in, U* out, int64_t count, int op, char* const* peers,
                       int world, int rank, int64_t setup_off, int64_t setup_bytes,
                       unsigned long long gen, cudaStream_t st) {
  xallreduce_kernel<U><<<1, 1024, 0, st>>>(in, out, count, op, peers, world, rank, setup_off,
                                           setup_bytes, gen);
  count_launch();
}
template void launch_xallreduce<float>(const float*, float*, int64_t, int, char* const*, int,
                                       int, int64_t, int64_t, unsigned long long, cudaStream_t);
template void launch_xallreduce<double>(const double*, double*, int64_t, int, char* const*, int,
                                        int, int64_t, int64_t, unsigned long long, cudaStream_t);
template void launch_xallreduce<int32_t>(const int32_t*, int32_t*, int64_t, int, char* const*,
                                         int, int, int64_t, int64_t, unsigned long long,
                                         cudaStream_t);

template <class T>
void launch_tail_finalize(const TailArgs<T>& t, const double* dpart, int grid, cudaStream_t st) {
  (void)dpart;
  (void)grid;
  tail_finalize_kernel<T><<<1, 32, 0, st>>>(t);
  count_launch();
}

template void launch_tail_finalize<float>(const TailArgs<float>&, const double*, int,
                                          cudaStream_t);
template void launch_tail_finalize<double>(const TailArgs<double>&, const double*, int,
                                           cudaStream_t);
template int tail_grid<float>(int);
template int tail_grid<double>(int);
template cudaError_t launch_tail<float>(const TailArgs<float>&, float*, double*, unsigned*, int,
                                        cudaStream_t);
template cudaError_t launch_tail<double>(const TailArgs<double>&, double*, double*, unsigned*,
                                         int, cudaStream_t);


}  // namespace drotb
