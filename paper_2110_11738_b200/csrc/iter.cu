// iter.cu -- KF: one launch per DROT iteration (fast reduction order, one
// GPU).  The fused sweep K1 (sweep.cuh) with the whole per-iteration tail
// of the solve loop folded into its prologue and epilogue:
//
//   prologue  phi_i = (ta_i + coef) * (1/n), varphi_j = (tb_j + coef) * (1/m)
//             (solver.hpp:279-285; ta = a - 2r and tb = b - 2s were formed by
//             the previous launch, coef is its Book value) for the CTA's rows
//             and columns; the CTAs of tile column 0 / tile row 0 also store
//             them and reduce the exact dual value and fixed-point partials
//             of the previous iteration (patched one iteration late, like the
//             cooperative tail's fused gate, tail.cu / gate.cuh)
//   sweep     K1 unchanged, except that varphi comes from shared memory and
//             the 64-row column sums are combined per CTA (vcta)
//   epilogue  "last arriving CTA" merges, no grid barrier and no co-residency
//             requirement:
//               column tile gc complete  -> v, s = v - q, tb, b -= s, record
//               (row block rb, u group) complete -> grouped row strip
//               row block rb complete    -> u, r = u - p, ta, a -= r, record
//               all records present      -> totals in fixed order, the
//                 recursions (merge_scalars), the pending patch and the fused
//                 gate on the Book (solver.hpp:266-289, 406-504)
//
// Every reduction runs in a fixed order independent of which CTA arrives
// last, so the iteration is deterministic.  A fired gate is confirmed by the
// exact matched-pair report in iter_confirm_kernel (launched after every
// iteration; it exits at once unless the gate fired), which evaluates phi /
// varphi on the fly.  iter_finalize_kernel materializes the pending duals
// and patches the last trace row at the end of a run.
//
// The tail this replaces (tail.cu) costs ~30 us per iteration at 10k^2 in
// grid barriers and launch gaps; here it overlaps the sweep except for the
// merges of the last column tile and row blocks.
#include <cmath>
#include <cstdint>

#include "drotb_internal.hpp"
#include "sweep.cuh"
#include "gate.cuh"

namespace drotb {

namespace {

constexpr int kNT = kWarpsPerCta * 32;  // K1 threads per CTA
constexpr int kCT = 256;                // confirm / finalize threads per CTA
constexpr int kCSlots = 16;

// fixed-order CTA sum of K values; every thread receives the totals
template <class U, int K>
__device__ __forceinline__ void cta_sum(U (&v)[K], U* sh /* K * nwarps */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh[k * nw + warp] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    U s = U(0);
    for (int w = 0; w < nw; ++w) s += sh[k * nw + w];
    v[k] = s;
  }
  __syncthreads();
}

template <class U>
__device__ __forceinline__ U cta_max(U v, U* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  U m = U(0);
  for (int w = 0; w < nw; ++w) m = fmax(m, sh[w]);
  __syncthreads();
  return m;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
// profiling aid (DROTB_TAIL_STAMPS=1): phase min / max timestamps
#define ITER_STAMP(slot, op)                                             \
  do {                                                                   \
    if (t.stamps && threadIdx.x == 0) op(t.stamps + (slot), gtimer());  \
  } while (0)

// arrival: one acq_rel fence, then relaxed atomics (several can be in
// flight); the last arriver fences again before reading the others' data
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned atom_add_relaxed(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
               : "memory");
  return old;
}

template <class T>
__device__ __forceinline__ T phi_of(T tv, T coef, T inv) {
  return (tv + coef) * inv;  // (a - 2r + coef) * inv_n, solver.hpp:280-285
}

// ---- epilogue merges -------------------------------------------------------
template <class T>
__device__ void merge_columns(const IterArgs<T>& g, int64_t gc, int64_t c0, int ncol,
                              double* shd, T* sht) {
  const TailArgs<T>& t = g.t;
  const int64_t n = g.pa.n;
  const int rbn = g.rbn;
  T s2 = T(0);
  double qb = 0.0, qs = 0.0;
  for (int cc = threadIdx.x; cc < ncol; cc += kNT) {
    const int64_t j = c0 + cc;
    T v = T(0);
    int r = 0;
    for (; r + 8 <= rbn; r += 8) {
      T x8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x8[k] = __ldcg(g.vcta + (r + k) * n + j);
#pragma unroll
      for (int k = 0; k < 8; ++k) v += x8[k];
    }
    for (; r < rbn; ++r) v += __ldcg(g.vcta + r * n + j);
    const T qj = t.q[j];
    const T s = v - qj;  // solver.hpp:271-272
    t.s_new[j] = s;
    const T bj = t.b[j];
    g.tb[j] = bj - T(2) * s;
    g.b_prev[j] = bj;
    t.b[j] = bj - s;  // solver.hpp:288
    s2 += s * s;
    qb += static_cast<double>(qj) * static_cast<double>(bj);
    qs += static_cast<double>(qj) * static_cast<double>(s);
  }
  // the K1 scalars of the column tile's rbn CTAs
  T c5[5] = {T(0), T(0), T(0), T(0), T(0)};  // cost, prev, dual, dx, #bad
  T mx = T(0);
  for (int r = threadIdx.x; r < rbn; r += kNT) {
    const PassPartial<T>* pp = g.pa.partials + gc * rbn + r;
    c5[0] += __ldcg(&pp->cost);
    c5[1] += __ldcg(&pp->prev);
    c5[2] += __ldcg(&pp->dual);
    c5[3] += __ldcg(&pp->dx);
    mx = fmax(mx, __ldcg(&pp->max_abs));
    c5[4] += __ldcg(&pp->bad) ? T(1) : T(0);
  }
  T t6[6] = {c5[0], c5[1], c5[2], c5[3], c5[4], s2};
  cta_sum<T, 6>(t6, sht);
  mx = cta_max<T>(mx, sht);
  double d2[2] = {qb, qs};
  cta_sum<double, 2>(d2, shd);
  if (threadIdx.x == 0) {
    IterColRec<T> rec;
    rec.cost = t6[0];
    rec.prev = t6[1];
    rec.dual = t6[2];
    rec.dx = t6[3];
    rec.mx = mx;
    rec.s2 = t6[5];
    rec.bad = t6[4] > T(0) ? 1 : 0;
    rec.pad = 0;
    rec.qb = d2[0];
    rec.qs = d2[1];
    g.colrec[gc] = rec;
    g.cnt[g.off_col + gc] = 0u;
  }
}

template <class T>
__device__ void merge_row_group(const IterArgs<T>& g, int64_t rb, int grp) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  const int64_t ld = g.pa.ld;
  const int64_t row0 = (rb * kNT + threadIdx.x) * R;
  if (row0 < g.pa.m) {
    const int g0 = grp * g.gu;
    const int g1 = min(g.gcn, g0 + g.gu);
    T acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = T(0);
    int s = g0;
    for (; s + 8 <= g1; s += 8) {
      V x8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        x8[q] = __ldcg(reinterpret_cast<const V*>(g.pa.ustrip + (s + q) * ld + row0));
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        T e[R];
        unpack(x8[q], e);
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] += e[k];
      }
    }
    for (; s < g1; ++s) {
      T e[R];
      unpack(__ldcg(reinterpret_cast<const V*>(g.pa.ustrip + s * ld + row0)), e);
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] += e[k];
    }
    *reinterpret_cast<V*>(g.ugrp + grp * ld + row0) = pack4(acc);
  }
  if (threadIdx.x == 0) g.cnt[g.off_ug + rb * g.ngrp + grp] = 0u;
}

template <class T>
__device__ void merge_rows(const IterArgs<T>& g, int64_t rb, double* shd, T* sht) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  const TailArgs<T>& t = g.t;
  const int64_t ld = g.pa.ld, m = g.pa.m;
  const int64_t row0 = (rb * kNT + threadIdx.x) * R;
  T sr = T(0), sr2 = T(0);
  double pa = 0.0, pr = 0.0;
  if (row0 < m) {
    T uu[R];
#pragma unroll
    for (int k = 0; k < R; ++k) uu[k] = T(0);
    int s = 0;
    for (; s + 8 <= g.ngrp; s += 8) {
      V x8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        x8[q] = __ldcg(reinterpret_cast<const V*>(g.ugrp + (s + q) * ld + row0));
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        T e[R];
        unpack(x8[q], e);
#pragma unroll
        for (int k = 0; k < R; ++k) uu[k] += e[k];
      }
    }
    for (; s < g.ngrp; ++s) {
      T e[R];
      unpack(__ldcg(reinterpret_cast<const V*>(g.ugrp + s * ld + row0)), e);
#pragma unroll
      for (int k = 0; k < R; ++k) uu[k] += e[k];
    }
    const int nvalid = static_cast<int>(imin64(R, m - row0));
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (k < nvalid) {
        const int64_t i = row0 + k;
        const T pi = t.p[i];
        const T r = uu[k] - pi;  // solver.hpp:269-270
        t.r_new[i] = r;
        const T ai = t.a[i];
        g.ta[i] = ai - T(2) * r;
        g.a_prev[i] = ai;
        t.a[i] = ai - r;  // solver.hpp:287
        sr += r;
        sr2 += r * r;
        pa += static_cast<double>(pi) * static_cast<double>(ai);
        pr += static_cast<double>(pi) * static_cast<double>(r);
      }
    }
  }
  T t2[2] = {sr, sr2};
  cta_sum<T, 2>(t2, sht);
  double d2[2] = {pa, pr};
  cta_sum<double, 2>(d2, shd);
  if (threadIdx.x == 0) {
    IterRowRec<T> rec;
    rec.sr = t2[0];
    rec.sr2 = t2[1];
    rec.pa = d2[0];
    rec.pr = d2[1];
    g.rowrec[rb] = rec;
    g.cnt[g.off_row + rb] = 0u;
  }
}

// all records present: totals, recursions, pending patch, fused gate
template <class T>
__device__ void iteration_final(const IterArgs<T>& g, double* shd, T* sht) {
  const TailArgs<T>& t = g.t;
  __shared__ Book<T> sbk;
  book_load(&sbk, t.book);
  ITER_STAMP(1, atomicMax);
  T t8[8] = {T(0), T(0), T(0), T(0), T(0), T(0), T(0), T(0)};  // cost prev dual dx bad sr sr2 s2
  T mx = T(0);
  double d12[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) d12[k] = 0.0;
  for (int c = threadIdx.x; c < g.gcn; c += kNT) {
    const IterColRec<T>* rc = g.colrec + c;
    t8[0] += __ldcg(&rc->cost);
    t8[1] += __ldcg(&rc->prev);
    t8[2] += __ldcg(&rc->dual);
    t8[3] += __ldcg(&rc->dx);
    t8[4] += __ldcg(&rc->bad) ? T(1) : T(0);
    t8[7] += __ldcg(&rc->s2);
    mx = fmax(mx, __ldcg(&rc->mx));
    d12[10] += __ldcg(&rc->qb);
    d12[11] += __ldcg(&rc->qs);
#pragma unroll
    for (int k = 0; k < 4; ++k) d12[4 + k] += __ldcg(g.ucol + c * 4 + k);
  }
  for (int r = threadIdx.x; r < g.rbn; r += kNT) {
    const IterRowRec<T>* rr = g.rowrec + r;
    t8[5] += __ldcg(&rr->sr);
    t8[6] += __ldcg(&rr->sr2);
    d12[8] += __ldcg(&rr->pa);
    d12[9] += __ldcg(&rr->pr);
#pragma unroll
    for (int k = 0; k < 4; ++k) d12[k] += __ldcg(g.urow + r * 4 + k);
  }
  cta_sum<T, 8>(t8, sht);
  mx = cta_max<T>(mx, sht);
  cta_sum<double, 12>(d12, shd);
  ITER_STAMP(2, atomicMax);
  if (threadIdx.x == 0) {
    // {cost, prev, dual, dx, max|t|, sum r, |r|^2, |s|^2} (merge_kernel order)
    const T tot[8] = {t8[0], t8[1], t8[2], t8[3], mx, t8[5], t8[6], t8[7]};
    merge_scalars<T>(&sbk, t, tot, t8[4] > T(0) ? 1 : 0);
    const double dp8[8] = {d12[0], d12[1], d12[2], d12[3], d12[4], d12[5], d12[6], d12[7]};
    patch_pending<T>(&sbk, t, dp8);  // the previous iteration's exact dual / trace terms
    if (!sbk.failed) {
      if (!sbk.stop) {
        const double coef = static_cast<double>(sbk.coef);
        const double inv_n = 1.0 / static_cast<double>(t.n_global);
        const double inv_m = 1.0 / static_cast<double>(t.m_global);
        const double dual_alg = ((d12[8] - 2.0 * d12[9] + coef * sbk.sum_p) * inv_n +
                                 (d12[10] - 2.0 * d12[11] + coef * sbk.sum_q) * inv_m) /
                                static_cast<double>(t.rho);
        gate_fused<T>(&sbk, t, dual_alg);
      }
      sbk.phi_mat = 0;  // phi_{k+1} pending in ta / tb / coef
    } else {
      sbk.phi_mat = 1;  // non-finite pass: the arrays hold phi_k, the state of solver.hpp:266
    }
  }
  ITER_STAMP(3, atomicMax);
  book_store(t.book, &sbk);
  ITER_STAMP(4, atomicMax);
  if (sbk.failed) {  // step_impl returns before a -= r, b -= s (solver.hpp:266)
    for (int64_t i = threadIdx.x; i < g.pa.m; i += kNT) t.a[i] = __ldcg(g.a_prev + i);
    for (int64_t j = threadIdx.x; j < g.pa.n; j += kNT) t.b[j] = __ldcg(g.b_prev + j);
  }
  if (threadIdx.x == 0) g.cnt[0] = 0u;
}

template <class T, int MODE, bool DUAL, bool DX>
__global__ void __launch_bounds__(kNT, DROTB_ASYNC_MINB) iter_kernel(const IterArgs<T> g) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  constexpr int ROWS_W = 32 * R;
  constexpr int NB = ROWS_W / kVBlockRows;
  const PassArgs<T>& a = g.pa;
  const TailArgs<T>& t = g.t;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ PassAcc<T> wacc[kWarpsPerCta];
  __shared__ double shd[12 * kWarpsPerCta];
  __shared__ T sht[8 * kWarpsPerCta];
  __shared__ int s_flag[4];
  Book<T>* bk = t.book;
  ITER_STAMP(0, atomicMin);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rb = blockIdx.x, gc = blockIdx.y;
  const int64_t c0 = gc * a.tc;
  const int64_t c1 = imin64(a.n, c0 + a.tc);
  const int ncol = static_cast<int>(c1 - c0);
  constexpr size_t ring_v = static_cast<size_t>(kAsyncS) * 2 * kAsyncG * 32;
  V* ring = reinterpret_cast<V*>(dyn_smem) + warp * ring_v;
  const int64_t wrow0 = (rb * kWarpsPerCta + warp) * ROWS_W;
  const int64_t row0 = wrow0 + static_cast<int64_t>(lane) * R;
  const int64_t nv = a.m - row0;
  const int nvalid = nv <= 0 ? 0 : (nv >= R ? R : static_cast<int>(nv));
  // the first column groups go in flight before the prologue's dependent
  // loads (reads only: harmless if the loop has stopped)
  ring_prime<T, MODE>(a, c0, c1, row0, nvalid > 0, ring, lane);
  const int stop = *reinterpret_cast<const volatile int*>(&bk->stop);
  const int pm = *reinterpret_cast<const volatile int*>(&bk->phi_mat);
  const T coef = *reinterpret_cast<const volatile T*>(&bk->coef);
  if (stop) {
    cp_async_wait<0>();
    return;
  }
  T* wbuf = reinterpret_cast<T*>(reinterpret_cast<V*>(dyn_smem) + kWarpsPerCta * ring_v) +
            warp * kChunkCols * ROWS_W;
  T* svphi = reinterpret_cast<T*>(dyn_smem + async_smem_bytes<T>());
  T* svs = svphi + a.tc;  // [kWarpsPerCta * NB][tc]

  // ---- prologue: the duals of this iteration ------------------------------
  const T inv_n = T(1) / static_cast<T>(t.n_global);
  const T inv_m = T(1) / static_cast<T>(t.m_global);
  const double drho = static_cast<double>(t.rho);
  double up[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // rows 0..3, columns 4..7
  for (int cc = tid; cc < ncol; cc += kNT) {
    const int64_t j = c0 + cc;
    T vp;
    if (pm) {
      vp = t.varphi[j];
    } else {
      vp = phi_of<T>(__ldcg(g.tb + j), coef, inv_m);
      if (rb == 0) {
        const T old = t.varphi[j];
        t.varphi[j] = vp;
        up[4] += static_cast<double>(t.q[j]) * static_cast<double>(vp) / drho;
        const double d = static_cast<double>(vp) - static_cast<double>(old);
        up[5] += d * d;
        up[6] += d;
        // s of the previous iteration is s_old here, the one before s_new
        up[7] += d * (static_cast<double>(t.s_old[j]) - static_cast<double>(t.s_new[j]));
      }
    }
    svphi[cc] = vp;
  }
  T ph[R], u[R];
#pragma unroll
  for (int k = 0; k < R; ++k) ph[k] = u[k] = T(0);
  if (nvalid > 0) {
    if (pm) {
      unpack(*reinterpret_cast<const V*>(t.phi + row0), ph);
    } else {
      T tv[R];
      unpack(__ldcg(reinterpret_cast<const V*>(g.ta + row0)), tv);
#pragma unroll
      for (int k = 0; k < R; ++k) ph[k] = k < nvalid ? phi_of<T>(tv[k], coef, inv_n) : T(0);
      if (gc == 0) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (k < nvalid) {
            const int64_t i = row0 + k;
            const T old = t.phi[i];
            t.phi[i] = ph[k];
            up[0] += static_cast<double>(t.p[i]) * static_cast<double>(ph[k]) / drho;
            const double d = static_cast<double>(ph[k]) - static_cast<double>(old);
            up[1] += d * d;
            up[2] += d;
            up[3] += d * (static_cast<double>(t.r_old[i]) - static_cast<double>(t.r_new[i]));
          }
        }
      }
    }
  }
  if (!pm && (gc == 0 || rb == 0)) {  // CTA-uniform
    cta_sum<double, 8>(up, shd);
    if (tid == 0) {
      if (gc == 0)
#pragma unroll
        for (int k = 0; k < 4; ++k) g.urow[rb * 4 + k] = up[k];
      if (rb == 0)
#pragma unroll
        for (int k = 0; k < 4; ++k) g.ucol[gc * 4 + k] = up[4 + k];
    }
  }
  __syncthreads();  // svphi

  // ---- the sweep (K1) -------------------------------------------------------
  PassAcc<T> acc{T(0), T(0), T(0), T(0), T(0), false};
  if (__all_sync(0xffffffffu, nvalid == R))
    pass_tile_async<T, MODE, DUAL, DX, false, true>(a, c0, c1, wrow0, row0, nvalid, ph, u, acc,
                                                    wbuf, ring, lane, svphi, svs, a.tc, warp);
  else
    pass_tile_async<T, MODE, DUAL, DX, true, true>(a, c0, c1, wrow0, row0, nvalid, ph, u, acc,
                                                   wbuf, ring, lane, svphi, svs, a.tc, warp);
  if (nvalid > 0) *reinterpret_cast<V*>(a.ustrip + gc * a.ld + row0) = pack4(u);
  acc.cost = warp_sum(acc.cost);
  acc.prev = warp_sum(acc.prev);
  acc.dual = warp_sum(acc.dual);
  acc.dx = warp_sum(acc.dx);
  acc.mx = warp_max(acc.mx);
  const bool wbad = __any_sync(0xffffffffu, acc.bad);
  if (lane == 0) {
    acc.bad = wbad;
    wacc[warp] = acc;
  }
  __syncthreads();
  if (tid == 0) {
    PassPartial<T> out{T(0), T(0), T(0), T(0), T(0), 0, 0};
#pragma unroll
    for (int w = 0; w < kWarpsPerCta; ++w) {
      out.cost += wacc[w].cost;
      out.prev += wacc[w].prev;
      out.dual += wacc[w].dual;
      out.dx += wacc[w].dx;
      out.max_abs = fmax(out.max_abs, wacc[w].mx);
      out.bad |= wacc[w].bad ? 1 : 0;
    }
    a.partials[gc * gridDim.x + rb] = out;  // column-tile major: the merge reads rbn in a row
  }
  // CTA-level column partials, 64-row blocks in ascending order
  for (int cc = tid; cc < ncol; cc += kNT) {
    T s = T(0);
#pragma unroll
    for (int w = 0; w < kWarpsPerCta * NB; ++w) s += svs[w * a.tc + cc];
    g.vcta[rb * a.n + c0 + cc] = s;
  }

  // ---- epilogue: arrivals and merges -------------------------------------
  __syncthreads();
  ITER_STAMP(7, atomicMax);
  if (tid == 0) {
    fence_acq_rel();
    const int grp = static_cast<int>(gc / g.gu);
    const int members = min(g.gu, g.gcn - grp * g.gu);
    const unsigned o0 = atom_add_relaxed(g.cnt + g.off_col + gc, 1u);
    const unsigned o1 = atom_add_relaxed(g.cnt + g.off_ug + rb * g.ngrp + grp, 1u);
    s_flag[0] = o0 == static_cast<unsigned>(g.rbn - 1);
    s_flag[1] = o1 == static_cast<unsigned>(members - 1);
    s_flag[2] = 0;
    if (s_flag[0] || s_flag[1]) fence_acq_rel();
  }
  __syncthreads();
  int arrivals = 0;
  if (s_flag[0]) {
    merge_columns<T>(g, gc, c0, ncol, shd, sht);
    ++arrivals;
  }
  if (s_flag[1]) {
    const int grp = static_cast<int>(gc / g.gu);
    merge_row_group<T>(g, rb, grp);
    __syncthreads();
    if (tid == 0) {
      fence_acq_rel();
      s_flag[2] = atom_add_relaxed(g.cnt + g.off_row + rb, 1u) == static_cast<unsigned>(g.ngrp - 1);
      if (s_flag[2]) fence_acq_rel();
    }
    __syncthreads();
    if (s_flag[2]) {
      merge_rows<T>(g, rb, shd, sht);
      ++arrivals;
    }
  }
  if (arrivals == 0) return;
  __syncthreads();
  if (tid == 0) {
    fence_acq_rel();
    const unsigned old = atom_add_relaxed(g.cnt, static_cast<unsigned>(arrivals));
    s_flag[3] = old + arrivals == static_cast<unsigned>(g.rbn + g.gcn);
    if (s_flag[3]) fence_acq_rel();
  }
  __syncthreads();
  if (!s_flag[3]) return;
  ITER_STAMP(5, atomicMax);
  iteration_final<T>(g, shd, sht);
  ITER_STAMP(6, atomicMax);
}

// ---- confirm: the exact matched-pair report when the gate fired ----------
// (solver.hpp:312-354, 503-519) with phi_{k+1} / varphi_{k+1} evaluated from
// ta / tb / coef, plus the exact dual value and fixed-point partials of the
// iteration (patched before the decision, as the cooperative tail does).
template <class T>
__global__ void __launch_bounds__(kCT) iter_confirm_kernel(const IterArgs<T> g) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  const TailArgs<T>& t = g.t;
  Book<T>* bk = t.book;
  if (!*reinterpret_cast<const volatile int*>(&bk->confirm) ||
      *reinterpret_cast<const volatile int*>(&bk->stop) == 1)
    return;
  __shared__ double shd[12 * (kCT / 32)];
  __shared__ int s_last;
  const int64_t m = g.pa.m, n = g.pa.n, ld = g.pa.ld;
  const int G = gridDim.x;
  const T coef = *reinterpret_cast<const volatile T*>(&bk->coef);
  const T inv_n = T(1) / static_cast<T>(t.n_global);
  const T inv_m = T(1) / static_cast<T>(t.m_global);
  const bool folded = *reinterpret_cast<const volatile int*>(&bk->folded) != 0;
  const double drho = static_cast<double>(t.rho);
  double part[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) part[k] = 0.0;
  // exact dual value and fixed-point terms (the update phase of tail.cu)
  const int64_t TT = static_cast<int64_t>(G) * kCT;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * kCT + threadIdx.x; idx < m + n;
       idx += TT) {
    if (idx < m) {
      const T ph = phi_of<T>(__ldcg(g.ta + idx), coef, inv_n);
      const double d = static_cast<double>(ph) - static_cast<double>(t.phi[idx]);
      part[0] += static_cast<double>(t.p[idx]) * static_cast<double>(ph) / drho;
      part[1] += d * d;
      part[2] += d;
      part[3] += d * (static_cast<double>(__ldcg(t.r_new + idx)) - static_cast<double>(t.r_old[idx]));
    } else {
      const int64_t j = idx - m;
      const T vp = phi_of<T>(__ldcg(g.tb + j), coef, inv_m);
      const double d = static_cast<double>(vp) - static_cast<double>(t.varphi[j]);
      part[4] += static_cast<double>(t.q[j]) * static_cast<double>(vp) / drho;
      part[5] += d * d;
      part[6] += d;
      part[7] += d * (static_cast<double>(__ldcg(t.s_new + j)) - static_cast<double>(t.s_old[j]));
    }
  }
  // the report sweep (tail.cu phase C)
  const int64_t ngx = (m + int64_t(kCT) * R - 1) / (int64_t(kCT) * R);
  const int64_t ncs = imin64(n, (2 * static_cast<int64_t>(G) + ngx - 1) / ngx);
  for (int64_t unit = blockIdx.x; unit < ngx * ncs; unit += G) {
    const int64_t rx = unit % ngx, cs = unit / ngx;
    const int64_t row0 = (rx * kCT + threadIdx.x) * R;
    if (row0 >= m) continue;
    const int nvalid = static_cast<int>(imin64(R, m - row0));
    double mu[R];
#pragma unroll
    for (int k = 0; k < R; ++k)
      mu[k] = k < nvalid
                  ? static_cast<double>(phi_of<T>(__ldcg(g.ta + row0 + k), coef, inv_n)) / drho
                  : 0.0;
    for (int64_t j = cs; j < n; j += ncs) {
      const double nu_j = static_cast<double>(phi_of<T>(__ldcg(g.tb + j), coef, inv_m)) / drho;
      T xv[R], cv[R];
      unpack(__ldcs(reinterpret_cast<const V*>(g.pa.xy + j * ld + row0)), xv);
      unpack(__ldcs(reinterpret_cast<const V*>(g.pa.cost + j * ld + row0)), cv);
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k < nvalid)
          report_elem_mu<T>(xv[k], cv[k], mu[k], nu_j, t.rho, folded, part[8], part[9]);
    }
  }
  cta_sum<double, 10>(part, shd);
  if (threadIdx.x < 10) g.dpart[blockIdx.x * kCSlots + threadIdx.x] = part[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(g.cnt + 1, 1u) == static_cast<unsigned>(G - 1);
    if (s_last) __threadfence();
  }
  __syncthreads();
  if (!s_last) return;
  double tot[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) tot[k] = 0.0;
  for (int b = threadIdx.x; b < G; b += kCT)
#pragma unroll
    for (int k = 0; k < 10; ++k) tot[k] += __ldcg(g.dpart + b * kCSlots + k);
  cta_sum<double, 10>(tot, shd);
  __shared__ Book<T> sbk;
  book_load(&sbk, bk);
  if (threadIdx.x == 0) {
    const double d8[8] = {tot[0], tot[1], tot[2], tot[3], tot[4], tot[5], tot[6], tot[7]};
    patch_pending<T>(&sbk, t, d8);  // exact dual value of this iteration
    report_decide<T>(&sbk, tot[8], tot[9], 0);
    g.cnt[1] = 0u;
  }
  book_store(bk, &sbk);
}

// ---- finalize: materialize pending duals, patch the last trace row -------
template <class T>
__global__ void __launch_bounds__(1024) iter_finalize_kernel(const IterArgs<T> g) {
  const TailArgs<T>& t = g.t;
  Book<T>* bk = t.book;
  if (*reinterpret_cast<const volatile int*>(&bk->phi_mat)) return;
  __shared__ double shd[8 * 32];
  const int64_t m = g.pa.m, n = g.pa.n;
  const int64_t it = *reinterpret_cast<const volatile int64_t*>(&bk->iter);
  // r / s of the last completed iteration and of the one before
  const T* rn = (it & 1) ? g.rbuf1 : g.rbuf0;
  const T* ro = (it & 1) ? g.rbuf0 : g.rbuf1;
  const T* sn = (it & 1) ? g.sbuf1 : g.sbuf0;
  const T* so = (it & 1) ? g.sbuf0 : g.sbuf1;
  const T coef = *reinterpret_cast<const volatile T*>(&bk->coef);
  const T inv_n = T(1) / static_cast<T>(t.n_global);
  const T inv_m = T(1) / static_cast<T>(t.m_global);
  const double drho = static_cast<double>(t.rho);
  double part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const T ph = phi_of<T>(g.ta[i], coef, inv_n);
    const T old = t.phi[i];
    t.phi[i] = ph;
    part[0] += static_cast<double>(t.p[i]) * static_cast<double>(ph) / drho;
    const double d = static_cast<double>(ph) - static_cast<double>(old);
    part[1] += d * d;
    part[2] += d;
    part[3] += d * (static_cast<double>(rn[i]) - static_cast<double>(ro[i]));
  }
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const T vp = phi_of<T>(g.tb[j], coef, inv_m);
    const T old = t.varphi[j];
    t.varphi[j] = vp;
    part[4] += static_cast<double>(t.q[j]) * static_cast<double>(vp) / drho;
    const double d = static_cast<double>(vp) - static_cast<double>(old);
    part[5] += d * d;
    part[6] += d;
    part[7] += d * (static_cast<double>(sn[j]) - static_cast<double>(so[j]));
  }
  cta_sum<double, 8>(part, shd);
  __shared__ Book<T> sbk;
  book_load(&sbk, bk);
  if (threadIdx.x == 0) {
    patch_pending<T>(&sbk, t, part);
    sbk.phi_mat = 1;
  }
  book_store(bk, &sbk);
}

template <class T, int MODE, bool DUAL, bool DX>
void launch_iter_t(const IterArgs<T>& g, cudaStream_t st) {
  static bool attr = [] {
    cudaFuncSetAttribute(iter_kernel<T, MODE, DUAL, DX>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(iter_smem_bytes<T>(256)));
    return true;
  }();
  (void)attr;
  dim3 grid(static_cast<unsigned>(g.rbn), static_cast<unsigned>(g.gcn));
  iter_kernel<T, MODE, DUAL, DX>
      <<<grid, kNT, iter_smem_bytes<T>(g.pa.tc), st>>>(g);
  count_launch();
}

}  // namespace

template <class T>
void iter_layout(int64_t m, int64_t n, int64_t tc, int32_t* rbn, int32_t* gcn, int32_t* gu,
                 int32_t* ngrp, int64_t* cnt_words) {
  constexpr int R = 16 / sizeof(T);
  const int64_t rows_cta = int64_t(kNT) * R;
  *rbn = static_cast<int32_t>((m + rows_cta - 1) / rows_cta);
  *gcn = static_cast<int32_t>((n + tc - 1) / tc);
  int32_t g = static_cast<int32_t>(std::ceil(std::sqrt(static_cast<double>(*gcn))));
  if (g < 1) g = 1;
  *gu = g;
  *ngrp = (*gcn + g - 1) / g;
  *cnt_words = 32 + *gcn + *rbn + static_cast<int64_t>(*rbn) * *ngrp;
}

template <class T>
size_t iter_smem_bytes(int64_t tc) {
  constexpr int R = 16 / sizeof(T);
  constexpr int NB = 32 * R / kVBlockRows;
  return async_smem_bytes<T>() +
         static_cast<size_t>(tc) * sizeof(T) * (1 + static_cast<size_t>(kWarpsPerCta) * NB);
}

template <class T>
void launch_iter(const IterArgs<T>& g, int mode, bool want_dual, bool want_dx, cudaStream_t st) {
#define DROTB_ITER_CASE(M)                                           \
  case M:                                                            \
    if (want_dual) {                                                 \
      if (want_dx) launch_iter_t<T, M, true, true>(g, st);           \
      else launch_iter_t<T, M, true, false>(g, st);                  \
    } else {                                                         \
      if (want_dx) launch_iter_t<T, M, false, true>(g, st);          \
      else launch_iter_t<T, M, false, false>(g, st);                 \
    }                                                                \
    break;
  switch (mode) {
    DROTB_ITER_CASE(kPlain0)
    DROTB_ITER_CASE(kPlain1)
    DROTB_ITER_CASE(kFold)
    default:
      launch_iter_t<T, kSkip, false, false>(g, st);
  }
#undef DROTB_ITER_CASE
}

template <class T>
void launch_iter_confirm(const IterArgs<T>& g, cudaStream_t st) {
  iter_confirm_kernel<T><<<kIterConfirmGrid, kCT, 0, st>>>(g);
  count_launch();
}

template <class T>
void launch_iter_finalize(const IterArgs<T>& g, cudaStream_t st) {
  iter_finalize_kernel<T><<<1, 1024, 0, st>>>(g);
  count_launch();
}

#define DROTB_ITER_INST(T)                                                                    \
  template void iter_layout<T>(int64_t, int64_t, int64_t, int32_t*, int32_t*, int32_t*,      \
                               int32_t*, int64_t*);                                           \
  template size_t iter_smem_bytes<T>(int64_t);                                                \
  template void launch_iter<T>(const IterArgs<T>&, int, bool, bool, cudaStream_t);            \
  template void launch_iter_confirm<T>(const IterArgs<T>&, cudaStream_t);                     \
  template void launch_iter_finalize<T>(const IterArgs<T>&, cudaStream_t);
DROTB_ITER_INST(float)
DROTB_ITER_INST(double)
#undef DROTB_ITER_INST

}  // namespace drotb
