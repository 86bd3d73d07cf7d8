// persistent.cu -- KP: the persistent solver kernel (fast reduction order,
// one GPU).  One cooperative launch runs up to `iters` complete DROT
// iterations of the solve loop (solver.hpp:406-521); the phases of an
// iteration are separated by grid-wide barriers instead of kernel
// boundaries:
//
//   P1 sweep    every CTA streams its fixed slice of X (and C) -- the fused
//               update of fused.hpp:244-289, same per-element arithmetic as
//               K1 -- and leaves u run partials, 512-row v partials and its
//               pass scalars (cost, prev, dual^2, dx^2, max|t|, non-finite)
//   -- barrier --
//   P2 merge    u -> r = u - p, v -> s = v - q, partial sum r, |r|^2, |s|^2
//               (fused.hpp:312-321; solver.hpp:269-272)
//   -- barrier --
//   P3 update   every CTA reduces the per-CTA partials in the same fixed
//               order (identical totals everywhere, no broadcast needed),
//               runs the scalar recursions (solver.hpp:273-277, 425-437) on
//               its shared-memory replica of the solver state, then
//               phi / varphi / a / b (solver.hpp:279-289) and the dual-value
//               and fixed-point partials
//   -- barrier --
//   P4 gate     totals -> gate (solver.hpp:443-504), replicated; when it
//               fires, the exact matched-pair report streams X and C
//               (solver.hpp:312-354, 503-519) -- one more barrier
//
// Three barriers per iteration replace the three kernel boundaries (merge,
// update, graph IF node) of the per-launch path; the state never leaves the
// device and the host only reads the stop flag between launches.
//
// The sweep slice of CTA b is the flat range [b*W/G, (b+1)*W/G) of the
// (row block, column) space, W = n_rb * n: one or two contiguous column
// segments of a 4-warp row block, so u accumulates in registers across the
// whole segment (~n_rb + G partials in total instead of one per tile) and
// the cp.async pipeline never restarts inside a segment.  Cross-CTA data is
// read with ld.global.cg (L2, coherent) -- L1 is not coherent across SMs.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstring>

#include "drotb_internal.hpp"
#include "sweep.cuh"

namespace drotb {

namespace cg = cooperative_groups;

namespace {

constexpr int kPT = kWarpsPerCta * 32;  // threads per CTA
constexpr int kPartStride = 16;         // per-CTA partial slots

// Grid-wide barrier of the cooperative launch.  cooperative_groups' grid
// sync measured 1.3-1.8 us on B200 at 148-592 CTAs against 2.3-3.1 us for a
// hand-rolled atomic counter + spin (scripts/barrier_bench.cu).
__device__ __forceinline__ void grid_barrier(unsigned* /*bar*/, unsigned /*nblocks*/) {
  cg::this_grid().sync();
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Sum over the G per-CTA partial slots [off, off+K) in a fixed order:
// thread t takes CTAs t, t+kPT, ..., then a fixed warp tree and the warps in
// order.  Every CTA runs the same instructions on the same data, so every
// CTA obtains bit-identical totals.  Result broadcast to all threads.
template <class U, int K>
__device__ __forceinline__ void cta_totals(const U* part, int nblocks, int off, U (&out)[K],
                                           U* sh /* K * kWarpsPerCta */) {
  U acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = U(0);
  for (int b = threadIdx.x; b < nblocks; b += kPT)
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] += __ldcg(part + b * kPartStride + off + k);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = warp_sum(acc[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh[k * kWarpsPerCta + warp] = acc[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    U s = U(0);
#pragma unroll
    for (int w = 0; w < kWarpsPerCta; ++w) s += sh[k * kWarpsPerCta + w];
    out[k] = s;
  }
  __syncthreads();
}

template <class T>
__device__ __forceinline__ T cta_max(const T* part, int nblocks, int off, T* sh) {
  T mx = T(0);
  for (int b = threadIdx.x; b < nblocks; b += kPT) mx = fmax(mx, __ldcg(part + b * kPartStride + off));
  mx = warp_max(mx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = mx;
  __syncthreads();
  T r = T(0);
#pragma unroll
  for (int w = 0; w < kWarpsPerCta; ++w) r = fmax(r, sh[w]);
  __syncthreads();
  return r;
}

// Block reduction of K values into the CTA's partial slots (fixed tree).
template <class U, int K>
__device__ __forceinline__ void cta_store(U (&v)[K], U* part, int off, U* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh[k * kWarpsPerCta + warp] = v[k];
  __syncthreads();
  if (threadIdx.x < K) {
    U s = U(0);
#pragma unroll
    for (int w = 0; w < kWarpsPerCta; ++w) s += sh[threadIdx.x * kWarpsPerCta + w];
    part[blockIdx.x * kPartStride + off + threadIdx.x] = s;
  }
  __syncthreads();
}

// P1 on one column segment [c0, c1) of row block rbk: the cp.async ring of
// K1-async over sub-segments of kSub columns.  Per sub-segment the CTA
// stages varphi[j] in shared memory once (one coalesced L2 read per column
// for the 4 warps, instead of a dependent L2 load per warp and column); the
// per-warp v partials of kVGroup consecutive 16-column chunks go to one half
// of a double-buffered shared array and are combined over the 4 warps (fixed
// order) after one __syncthreads per kVGroup chunks, into vstrip[rbk][j].
constexpr int kVGroup = 4;

template <class T>
constexpr int sub_cols() {
  return 4096 / static_cast<int>(sizeof(T));  // 1024 fp32 / 512 fp64 columns
}

template <class T>
struct SweepSmem {
  T vp[sub_cols<T>()];                                      // staged varphi
  T vacc[2][kVGroup][kWarpsPerCta][kChunkCols];             // v partials
};

template <class T>
__device__ __forceinline__ void flush_vgroup(const PersistArgs<T>& g, SweepSmem<T>& sm, int half,
                                             int64_t rbk, int64_t l0, int64_t l1, int n_in,
                                             int64_t cbase, int64_t cstride, int64_t n) {
  // threads 0 .. kVGroup*16-1: one column of the group each
  const int t = threadIdx.x;
  if (t < kVGroup * kChunkCols) {
    const int ch = t / kChunkCols, c = t % kChunkCols;
    const int64_t l = l0 + static_cast<int64_t>(ch) * kChunkCols + c;
    if (ch < n_in && l < l1) {
      T tot = T(0);
#pragma unroll
      for (int w = 0; w < kWarpsPerCta; ++w) tot += sm.vacc[half][ch][w][c];
      g.vstrip[rbk * n + cbase + l * cstride] = tot;
    }
  }
}

// P1 over the local steps [l0, l1) of one row block: step l is column
// cbase + l * cstride (stride 1: a contiguous segment; stride k: the
// interleaved schedule, where the k CTAs of a row block take every k-th
// column so that co-running CTAs stream whole contiguous column bands).
template <class T, int MODE, bool DUAL, bool DX, bool MASK>
__device__ __forceinline__ void sweep_segment(const PersistArgs<T>& g, const PassArgs<T>& a,
                                              int64_t rbk, int64_t l0, int64_t l1,
                                              int64_t cbase, int64_t cstride, int64_t row0,
                                              int nvalid, const T (&ph)[16 / sizeof(T)],
                                              T (&u)[16 / sizeof(T)], PassAcc<T>& acc,
                                              T* wbuf, typename V16<T>::type* ring,
                                              SweepSmem<T>& sm, int warp, int lane) {
  constexpr int R = 16 / sizeof(T);
  constexpr int ROWS_W = 32 * R;
  constexpr int NB = ROWS_W / kVBlockRows;  // 64-row blocks per warp (2 fp32, 1 fp64)
  constexpr bool RC = MODE != kSkip;
  constexpr int S = kAsyncS, G = RC ? kAsyncG : 2 * kAsyncG, CH = kChunkCols;
  constexpr int NG = CH / G;
  constexpr int SUB = sub_cols<T>();
  static_assert(NG % S == 0, "stages must divide the groups of a chunk");
  static_assert(SUB % (CH * kVGroup) == 0, "sub-segments hold whole chunk groups");
  const bool live = !MASK || nvalid > 0;
  auto xslot = [&](int st, int k) { return ring + (st * 2 * kAsyncG + k) * 32 + lane; };
  auto cslot = [&](int st, int k) {
    return ring + (st * 2 * kAsyncG + kAsyncG + k) * 32 + lane;
  };
  int half = 0;
  for (int64_t s0 = l0; s0 < l1; s0 += SUB) {
    const int64_t s1 = imin64(l1, s0 + SUB);
    __syncthreads();  // previous sub-segment's readers of sm.vp are done
    for (int64_t l = s0 + threadIdx.x; l < s1; l += kPT)
      sm.vp[l - s0] = __ldcg(a.varphi + cbase + l * cstride);
    __syncthreads();
    auto issue = [&](int st, int64_t lg) {
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int64_t l = lg + k;
        if (live && l < s1) {
          const int64_t off = (cbase + l * cstride) * a.ld + row0;
          cp_async16(xslot(st, k), a.xy + off);
          if (RC) cp_async16(cslot(st, k), a.cost + off);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int st = 0; st < S - 1; ++st) issue(st, s0 + st * G);
    int ch_in = 0;  // chunk index within the current v group
    int64_t gl0 = s0;
    for (int64_t j0 = s0; j0 < s1; j0 += CH) {
#pragma unroll
      for (int gg = 0; gg < NG; ++gg) {
        const int st = gg % S;
        issue((gg + S - 1) % S, j0 + (gg + S - 1) * G);
        cp_async_wait<S - 1>();
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int64_t l = j0 + gg * G + k;
          if (l < s1) {
            T x[R], cc[R];
#pragma unroll
            for (int t = 0; t < R; ++t) x[t] = cc[t] = T(0);
            if (live) {
              unpack(*xslot(st, k), x);
              if (RC) unpack(*cslot(st, k), cc);
            }
            compute_col<T, MODE, DUAL, DX, MASK>(a, x, cc, sm.vp[l - s0], cbase + l * cstride,
                                                 gg * G + k, row0, nvalid, ph, u, acc, wbuf,
                                                 lane);
          }
        }
      }
      const int cnt = static_cast<int>(imin64(CH, s1 - j0));
      __syncwarp();
      // per-warp column partials: lane (c, b) sums 64-row block b of staged
      // column c in row order, then the warp's blocks are added
      T sv = T(0);
      if (lane < CH * NB) {
        const int c = lane % CH, bb = lane / CH;
        if (c < cnt) {
          using V = typename V16<T>::type;
          const V* col = reinterpret_cast<const V*>(wbuf) + c * 32;
          const int g7 = c & 7;
          constexpr int QB = kVBlockRows / R;
#pragma unroll
          for (int qq = 0; qq < QB; ++qq) {
            T v4[R];
            unpack(col[(bb * QB + qq) ^ g7], v4);
#pragma unroll
            for (int t = 0; t < R; ++t) sv += v4[t];
          }
        }
      }
      if (NB == 2) sv += __shfl_down_sync(0xffffffffu, sv, 16);
      if (lane < CH) sm.vacc[half][ch_in][warp][lane] = sv;
      __syncwarp();  // the staging buffer is rewritten by the next chunk
      if (++ch_in == kVGroup || j0 + CH >= s1) {
        __syncthreads();
        flush_vgroup(g, sm, half, rbk, gl0, s1, ch_in, cbase, cstride, a.n);
        half ^= 1;
        ch_in = 0;
        gl0 = j0 + CH;
      }
    }
    cp_async_wait<0>();
  }
}

template <class T, int MODE, bool DUAL, bool DX, bool MASK>
__device__ __forceinline__ void sweep_rows(const PersistArgs<T>& g, const PassArgs<T>& a,
                                           int64_t rbk, int64_t l0, int64_t l1, int64_t cbase,
                                           int64_t cstride, int64_t slot, PassAcc<T>& acc,
                                           T* wbuf, typename V16<T>::type* ring,
                                           SweepSmem<T>& sm, int warp, int lane) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  constexpr int ROWS_W = 32 * R;
  const int64_t row0 = rbk * g.rows_cta + static_cast<int64_t>(warp) * ROWS_W +
                       static_cast<int64_t>(lane) * R;
  const int64_t nv = a.m - row0;
  const int nvalid = nv <= 0 ? 0 : (nv >= R ? R : static_cast<int>(nv));
  T ph[R], u[R];
  if (nvalid > 0) {
    unpack(__ldcg(reinterpret_cast<const V*>(a.phi + row0)), ph);
  } else {
#pragma unroll
    for (int t = 0; t < R; ++t) ph[t] = T(0);
  }
#pragma unroll
  for (int t = 0; t < R; ++t) u[t] = T(0);
  sweep_segment<T, MODE, DUAL, DX, MASK>(g, a, rbk, l0, l1, cbase, cstride, row0, nvalid, ph,
                                         u, acc, wbuf, ring, sm, warp, lane);
  if (nvalid > 0)
    *reinterpret_cast<V*>(g.ustrip + slot * g.rows_cta + (row0 - rbk * g.rows_cta)) = pack4(u);
}

template <class T, int MODE, bool DUAL, bool DX>
__device__ void sweep_phase(const PersistArgs<T>& g, const PassArgs<T>& a, int64_t f0,
                            int64_t f1, PassAcc<T>& acc, T* wbuf,
                            typename V16<T>::type* ring, SweepSmem<T>& sm, int warp,
                            int lane) {
  const int64_t n = a.n;
  if (g.ileave > 0) {
    // interleaved: CTA b < n_rb * k owns row block b % n_rb and the columns
    // j = b / n_rb (mod k); CTAs beyond n_rb * k only join the other phases
    const int64_t k = g.ileave;
    if (static_cast<int64_t>(blockIdx.x) >= g.n_rb * k) return;
    const int64_t rbk = blockIdx.x % g.n_rb, cg = blockIdx.x / g.n_rb;
    const int64_t ns = (n - cg + k - 1) / k;
    const bool full = (rbk + 1) * g.rows_cta <= a.m;
    if (full)
      sweep_rows<T, MODE, DUAL, DX, false>(g, a, rbk, 0, ns, cg, k, blockIdx.x, acc, wbuf,
                                           ring, sm, warp, lane);
    else
      sweep_rows<T, MODE, DUAL, DX, true>(g, a, rbk, 0, ns, cg, k, blockIdx.x, acc, wbuf, ring,
                                          sm, warp, lane);
    return;
  }
  int seg = 0;
  while (f0 < f1) {
    const int64_t rbk = f0 / n;
    const int64_t c0 = f0 - rbk * n;
    const int64_t c1 = imin64(n, c0 + (f1 - f0));
    const int64_t slot = static_cast<int64_t>(blockIdx.x) * g.max_seg + seg;
    const bool full = (rbk + 1) * g.rows_cta <= a.m;
    if (full)
      sweep_rows<T, MODE, DUAL, DX, false>(g, a, rbk, c0, c1, 0, 1, slot, acc, wbuf, ring, sm,
                                           warp, lane);
    else
      sweep_rows<T, MODE, DUAL, DX, true>(g, a, rbk, c0, c1, 0, 1, slot, acc, wbuf, ring, sm,
                                          warp, lane);
    f0 += c1 - c0;
    ++seg;
  }
}

template <class T>
__device__ __forceinline__ void tail_args_for(TailArgs<T>& tl, const PersistArgs<T>& g,
                                              int mode, bool folded_after, bool dx) {
  memset(&tl, 0, sizeof(tl));
  tl.m = g.pa.m;
  tl.n = g.pa.n;
  tl.m_global = g.m_global;
  tl.n_global = g.n_global;
  tl.folded_after = folded_after ? 1 : 0;
  tl.rho = g.pa.rho;
  tl.reads_cost = mode != kSkip;
  tl.want_dual = 1;
  tl.want_dx = dx ? 1 : 0;
  tl.solver = 1;
  tl.trace = blockIdx.x == 0 ? g.trace : nullptr;
}

template <class T, bool DX>
__global__ void __launch_bounds__(kPT, 3) solve_kernel(const PersistArgs<T> g) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  constexpr int ROWS_W = 32 * R;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ Book<T> S;
  __shared__ SweepSmem<T> sm;
  __shared__ PassAcc<T> wacc[kWarpsPerCta];
  __shared__ T shT[16 * kWarpsPerCta];
  __shared__ double shD[16 * kWarpsPerCta];
  __shared__ T mred[kWarpsPerCta][32];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned G = gridDim.x;
  constexpr size_t ring_v = static_cast<size_t>(kAsyncS) * 2 * kAsyncG * 32;  // V per warp
  V* ring = reinterpret_cast<V*>(dyn_smem) + warp * ring_v;
  T* wbuf = reinterpret_cast<T*>(reinterpret_cast<V*>(dyn_smem) + kWarpsPerCta * ring_v) +
            warp * kChunkCols * ROWS_W;

  if (tid == 0) S = *g.book;
  __syncthreads();
  if (S.stop) return;

  const PassArgs<T>& a = g.pa;
  const int64_t m = a.m, n = a.n;
  const int64_t W = g.n_rb * n;
  const int64_t f0 = static_cast<int64_t>(blockIdx.x) * W / G;
  const int64_t f1 = static_cast<int64_t>(blockIdx.x + 1) * W / G;
  const int64_t gt = static_cast<int64_t>(blockIdx.x) * kPT + tid;
  const int64_t TT = static_cast<int64_t>(G) * kPT;
  const T inv_n = T(1) / static_cast<T>(g.n_global);
  const T inv_m = T(1) / static_cast<T>(g.m_global);
  const double drho = static_cast<double>(a.rho);
  const bool fp = S.record_trace != 0;
  unsigned long long t_sweep = 0;

  for (int64_t it = 0; it < g.iters; ++it) {
    const int64_t k = S.iter;
    const bool folded = S.folded != 0;
    int mode;
    bool folded_after;
    if (g.engine_ref) {
      mode = (k & 1) ? kPlain1 : kPlain0;
      folded_after = false;
    } else if (g.skip_cost) {
      mode = folded ? kSkip : kFold;
      folded_after = !folded;
    } else {
      mode = (k & 1) ? kPlain1 : kPlain0;
      folded_after = folded;
    }
    const unsigned long long t0 = (blockIdx.x == 0 && tid == 0) ? globaltimer() : 0ull;

    // ---- P1: sweep -------------------------------------------------------
    PassAcc<T> acc{T(0), T(0), T(0), T(0), T(0), false};
    switch (mode) {
      case kPlain0:
        sweep_phase<T, kPlain0, true, DX>(g, a, f0, f1, acc, wbuf, ring, sm, warp, lane);
        break;
      case kPlain1:
        sweep_phase<T, kPlain1, true, DX>(g, a, f0, f1, acc, wbuf, ring, sm, warp, lane);
        break;
      case kFold:
        sweep_phase<T, kFold, true, DX>(g, a, f0, f1, acc, wbuf, ring, sm, warp, lane);
        break;
      default:
        sweep_phase<T, kSkip, false, false>(g, a, f0, f1, acc, wbuf, ring, sm, warp, lane);
    }
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
      T o[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int w = 0; w < kWarpsPerCta; ++w) {
        o[0] += wacc[w].cost;
        o[1] += wacc[w].prev;
        o[2] += wacc[w].dual;
        o[3] += wacc[w].dx;
        o[4] = fmax(o[4], wacc[w].mx);
        o[5] += wacc[w].bad ? T(1) : T(0);
      }
#pragma unroll
      for (int q = 0; q < 6; ++q) g.cpart[blockIdx.x * kPartStride + q] = o[q];
    }
    grid_barrier(g.bar, G);
    if (blockIdx.x == 0 && tid == 0) t_sweep += globaltimer() - t0;

    // ---- P2: merge -------------------------------------------------------
    T* r_new = (k & 1) ? g.rb0 : g.rb1;
    T* s_new = (k & 1) ? g.sb0 : g.sb1;
    const T* r_old = (k & 1) ? g.rb1 : g.rb0;
    const T* s_old = (k & 1) ? g.sb1 : g.sb0;
    {
      // groups of 32 consecutive rows (then columns), one group per CTA at a
      // time; warp w sums partials w, w+4, ... of the 32 indices (coalesced
      // 128-B loads), the 4 warp sums are added in warp order
      T pr[3] = {T(0), T(0), T(0)};
      const int64_t ngr = (m + 31) / 32, ngc = (n + 31) / 32;
      for (int64_t grp = blockIdx.x; grp < ngr + ngc; grp += G) {
        T acc = T(0);
        if (grp < ngr) {
          const int64_t idx = grp * 32 + lane;
          const int64_t rbk = (grp * 32) / g.rows_cta;  // 32 | rows_cta: one row block
          const int64_t li = idx - rbk * g.rows_cta;
          const int s1 = g.seg_ptr[rbk + 1];
          if (idx < m) {
            int s = g.seg_ptr[rbk] + warp;
            for (; s + 3 * kWarpsPerCta < s1; s += 4 * kWarpsPerCta) {
              T v4[4];
#pragma unroll
              for (int q = 0; q < 4; ++q)
                v4[q] = __ldcg(g.ustrip +
                               static_cast<int64_t>(g.seg_slot[s + q * kWarpsPerCta]) * g.rows_cta + li);
#pragma unroll
              for (int q = 0; q < 4; ++q) acc += v4[q];
            }
            for (; s < s1; s += kWarpsPerCta)
              acc += __ldcg(g.ustrip + static_cast<int64_t>(g.seg_slot[s]) * g.rows_cta + li);
          }
        } else {
          const int64_t j = (grp - ngr) * 32 + lane;
          if (j < n) {
            int64_t q0 = warp;
            for (; q0 + 3 * kWarpsPerCta < g.n_rb; q0 += 4 * kWarpsPerCta) {
              T v4[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) v4[q] = __ldcg(g.vstrip + (q0 + q * kWarpsPerCta) * n + j);
#pragma unroll
              for (int q = 0; q < 4; ++q) acc += v4[q];
            }
            for (; q0 < g.n_rb; q0 += kWarpsPerCta) acc += __ldcg(g.vstrip + q0 * n + j);
          }
        }
        mred[warp][lane] = acc;
        __syncthreads();
        if (warp == 0) {
          T tot = T(0);
#pragma unroll
          for (int w = 0; w < kWarpsPerCta; ++w) tot += mred[w][lane];
          if (grp < ngr) {
            const int64_t idx = grp * 32 + lane;
            if (idx < m) {
              const T r = tot - g.p[idx];
              r_new[idx] = r;
              pr[0] += r;
              pr[1] += r * r;
            }
          } else {
            const int64_t j = (grp - ngr) * 32 + lane;
            if (j < n) {
              const T sv = tot - g.q[j];
              s_new[j] = sv;
              pr[2] += sv * sv;
            }
          }
        }
        __syncthreads();
      }
      cta_store<T, 3>(pr, g.cpart, 6, shT);
    }
    grid_barrier(g.bar, G);

    // ---- P3: totals, scalar recursions, phi / varphi update ---------------
    {
      T t8[8];
      T s7[7];
      cta_totals<T, 7>(g.cpart, G, 0, s7, shT);  // cost prev dual dx max(ignored) bad sum_r
      T s2[2];
      cta_totals<T, 2>(g.cpart, G, 7, s2, shT);  // |r|^2 |s|^2
      const T mx = cta_max<T>(g.cpart, G, 4, shT);
      t8[0] = s7[0];
      t8[1] = s7[1];
      t8[2] = s7[2];
      t8[3] = s7[3];
      t8[4] = mx;
      t8[5] = s7[6];
      t8[6] = s2[0];
      t8[7] = s2[1];
      // slot 5 (bad count) and 6 (sum r) come from s7[5], s7[6]
      const int bad = s7[5] > T(0) ? 1 : 0;
      if (tid == 0) {
        TailArgs<T> tl;
        tail_args_for(tl, g, mode, folded_after, DX);
        merge_scalars<T>(&S, tl, t8, bad);
      }
      __syncthreads();
      if (S.failed) break;
    }
    {
      const T coef = S.coef;
      double part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int64_t idx = gt; idx < m + n; idx += TT) {
        if (idx < m) {
          const T r = __ldcg(r_new + idx);
          const T ph_old = __ldcg(a.phi + idx);
          const T ai = __ldcg(g.a + idx);
          const T ph = (ai - T(2) * r + coef) * inv_n;  // solver.hpp:280-282
          const_cast<T*>(a.phi)[idx] = ph;
          g.a[idx] = ai - r;  // solver.hpp:287
          part[0] = part[0] + static_cast<double>(g.p[idx]) * static_cast<double>(ph) / drho;
          g.mud[idx] = static_cast<double>(ph) / drho;  // mu_i of the confirm report
          if (fp) {
            const double d = static_cast<double>(ph) - static_cast<double>(ph_old);
            part[1] += d * d;
            part[2] += d;
            part[3] += d * (static_cast<double>(r) - static_cast<double>(__ldcg(r_old + idx)));
          }
        } else {
          const int64_t j = idx - m;
          const T s = __ldcg(s_new + j);
          const T vp_old = __ldcg(a.varphi + j);
          const T bj = __ldcg(g.b + j);
          const T vp = (bj - T(2) * s + coef) * inv_m;  // solver.hpp:283-285
          const_cast<T*>(a.varphi)[j] = vp;
          g.b[j] = bj - s;  // solver.hpp:288
          part[4] = part[4] + static_cast<double>(g.q[j]) * static_cast<double>(vp) / drho;
          if (fp) {
            const double d = static_cast<double>(vp) - static_cast<double>(vp_old);
            part[5] += d * d;
            part[6] += d;
            part[7] += d * (static_cast<double>(s) - static_cast<double>(__ldcg(s_old + j)));
          }
        }
      }
      cta_store<double, 8>(part, g.dpart, 0, shD);
    }
    grid_barrier(g.bar, G);

    // ---- P4: gate (+ exact confirm report) --------------------------------
    {
      double d8[8];
      cta_totals<double, 8>(g.dpart, G, 0, d8, shD);
      if (tid == 0) {
        TailArgs<T> tl;
        tail_args_for(tl, g, mode, folded_after, DX);
        gate_logic<T>(&S, tl, d8[0] + d8[4], d8[1], d8[2], d8[5], d8[6], d8[3] + d8[7]);
      }
      __syncthreads();
    }
    if (S.confirm && S.stop != 1) {
      // state_report of (X_{k+1}, phi/rho, varphi/rho) (solver.hpp:312-354)
      const bool fo = S.folded != 0;
      double part[2] = {0, 0};
      for (int64_t j = blockIdx.x; j < n; j += G) {
        const double nu_j = static_cast<double>(__ldcg(a.varphi + j)) / drho;
        const T* xc = a.xy + j * a.ld;
        const T* cc = a.cost + j * a.ld;
        for (int64_t i = tid; i < m; i += kPT)
          report_elem_mu<T>(__ldcg(xc + i), __ldcg(cc + i), __ldcg(g.mud + i), nu_j, a.rho, fo,
                            part[0], part[1]);
      }
      cta_store<double, 2>(part, g.dpart, 8, shD);
      grid_barrier(g.bar, G);
      double d2[2];
      cta_totals<double, 2>(g.dpart, G, 8, d2, shD);
      if (tid == 0) report_decide<T>(&S, d2[0], d2[1], 0);
      __syncthreads();
    }
    if (S.stop) break;
  }
  if (blockIdx.x == 0 && tid == 0) {
    *g.book = S;
    if (g.sweep_ns) *g.sweep_ns += t_sweep;
  }
}

}  // namespace

template <class T>
size_t persistent_smem_bytes() {
  return async_smem_bytes<T>();
}

template <class T>
int persistent_grid(int device) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const size_t smem = persistent_smem_bytes<T>();
  cudaFuncSetAttribute(solve_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  cudaFuncSetAttribute(solve_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  int p1 = 0, p2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, solve_kernel<T, true>, kPT, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, solve_kernel<T, false>, kPT, smem);
  per = p1 < p2 ? p1 : p2;
  return sms * per;
}

template <class T>
int rows_per_cta() {
  return kWarpsPerCta * 32 * (16 / static_cast<int>(sizeof(T)));
}

template <class T>
cudaError_t launch_persistent(const PersistArgs<T>& g, int grid, bool dx, cudaStream_t st) {
  const size_t smem = persistent_smem_bytes<T>();
  void* args[] = {const_cast<PersistArgs<T>*>(&g)};
  cudaError_t e;
  if (dx)
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(solve_kernel<T, true>),
                                    dim3(grid), dim3(kPT), args, smem, st);
  else
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(solve_kernel<T, false>),
                                    dim3(grid), dim3(kPT), args, smem, st);
  count_launch();
  return e;
}

template size_t persistent_smem_bytes<float>();
template size_t persistent_smem_bytes<double>();
template int persistent_grid<float>(int);
template int persistent_grid<double>(int);
template int rows_per_cta<float>();
template int rows_per_cta<double>();
template cudaError_t launch_persistent<float>(const PersistArgs<float>&, int, bool, cudaStream_t);
template cudaError_t launch_persistent<double>(const PersistArgs<double>&, int, bool,
                                               cudaStream_t);

}  // namespace drotb
