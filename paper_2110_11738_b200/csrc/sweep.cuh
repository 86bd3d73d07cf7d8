// sweep.cuh -- device building blocks of the fused DROT sweep (K1), shared
// by the per-launch kernels (kernels.cu) and the persistent solver kernel
// (persistent.cu).  See kernels.cu for the arithmetic contract.
#pragma once

#include <cfloat>
#include <cstdint>

#include "drotb_internal.hpp"

namespace drotb {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) {
  return a < b ? a : b;
}

template <class T>
struct V16;
template <>
struct V16<float> {
  using type = float4;
};
template <>
struct V16<double> {
  using type = double2;
};

__device__ __forceinline__ void unpack(const float4& v, float* o) {
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void unpack(const double2& v, double* o) {
  o[0] = v.x; o[1] = v.y;
}
__device__ __forceinline__ float4 pack4(const float* o) {
  return make_float4(o[0], o[1], o[2], o[3]);
}
__device__ __forceinline__ double2 pack4(const double* o) {
  return make_double2(o[0], o[1]);
}
template <class T>
__device__ __forceinline__ typename V16<T>::type vzero() {
  typename V16<T>::type z;
  T* p = reinterpret_cast<T*>(&z);
#pragma unroll
  for (int t = 0; t < int(16 / sizeof(T)); ++t) p[t] = T(0);
  return z;
}

// the per-iteration strips / partials K1 writes for the tail: evict_last
// keeps them in L2 while the sweep streams (PassArgs::l2hint bit 1)
__device__ __forceinline__ uint64_t keep_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_keep(float* p, float v, int hint) {
  if (hint & 2)
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(keep_policy())
                 : "memory");
  else
    *p = v;
}
__device__ __forceinline__ void st_keep(double* p, double v, int hint) {
  if (hint & 2)
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(keep_policy())
                 : "memory");
  else
    *p = v;
}
__device__ __forceinline__ void st_keep(float4* p, float4 v, int hint) {
  if (hint & 2)
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(keep_policy())
                 : "memory");
  else
    *p = v;
}
__device__ __forceinline__ void st_keep(double2* p, double2 v, int hint) {
  if (hint & 2)
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x),
                 "d"(v.y), "l"(keep_policy())
                 : "memory");
  else
    *p = v;
}
// loads of the small per-iteration vectors with the same evict_last policy
// (cg: data written by other CTAs of the same kernel)
__device__ __forceinline__ float ld_keep(const float* p) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(keep_policy()));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(keep_policy()));
  return v;
}
__device__ __forceinline__ float ld_keep_cg(const float* p) {
  float v;
  asm volatile("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(keep_policy()));
  return v;
}
__device__ __forceinline__ double ld_keep_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(keep_policy()));
  return v;
}

__device__ __forceinline__ float ld_keep_nc(const float* p) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(keep_policy()));
  return v;
}
__device__ __forceinline__ double ld_keep_nc(const double* p) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(keep_policy()));
  return v;
}
__device__ __forceinline__ float4 ld_keep(const float4* p) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(keep_policy()));
  return v;
}
__device__ __forceinline__ double2 ld_keep(const double2* p) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(keep_policy()));
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// one timeline point (min and max over the CTAs that record it)
__device__ __forceinline__ void timeline_point(unsigned long long* st, int64_t iter, int pt,
                                               unsigned long long t) {
  unsigned long long* w = st + ((iter & (kStampSlots - 1)) * kStampPts + pt) * 2;
  atomicMin(w, t);
  atomicMax(w + 1, t);
}

template <class T>
struct PassPartial;
// per-CTA K1 scalars, kept in L2 for the tail
template <class T>
__device__ __forceinline__ void st_partial_keep(PassPartial<T>* d, const PassPartial<T>& v) {
  st_keep(&d->cost, v.cost, 2);
  st_keep(&d->prev, v.prev, 2);
  st_keep(&d->dual, v.dual, 2);
  st_keep(&d->dx, v.dx, 2);
  st_keep(&d->max_abs, v.max_abs, 2);
  d->bad = v.bad;
}

template <class T>
__device__ __forceinline__ T max_finite();
template <>
__device__ __forceinline__ float max_finite<float>() { return FLT_MAX; }
template <>
__device__ __forceinline__ double max_finite<double>() { return DBL_MAX; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-shape block tree reduction of K values (deterministic: the tree
// depends only on blockDim).  Result valid in thread 0.
template <class T, int K>
__device__ __forceinline__ void block_sum(T (&v)[K], T* sh /* K*32 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh[k * 32 + warp] = v[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      T x = lane < nw ? sh[k * 32 + lane] : T(0);
      v[k] = warp_sum(x);
    }
  }
  __syncthreads();
}

// Grid-level "last block done" ticket (threadFenceReduction pattern).
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(ticket, 1u);
    is_last = (t == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// ---------------------------------------------------------------------------
// K1: the fused sweep
// ---------------------------------------------------------------------------
// Thread mapping: a warp owns 32*R consecutive rows (R = 16 B / sizeof(T)
// rows per lane, one 128-bit load per column) of one tile column
// [c0, c0+tc).  Each lane walks the tile's columns in order, so its row
// partials are exactly the reference's u strips (fused.hpp:267, tile-local
// running sum from 0).  Column partials must be sequential over each
// 64-row block (fused.hpp:268): the warp stages x+ of 16 columns in shared
// memory and one lane per (column, 64-row block) sums the 64 values in row
// order with 128-bit shared loads.
//
// Staging layout (per warp, 16 columns x 32R rows, 16-B chunks): chunk q
// (rows qR..qR+R-1) of column c lives at chunk slot c*32 + (q ^ (c & 7)).
// The STS.128 of a column (lane l writes chunk l) and the LDS.128 of the
// row-order reads (lane = column [+16 * block], same q across lanes) both
// touch 8 distinct 16-B bank groups per 8-lane phase: conflict free.
//
// Memory pipeline: columns are processed in groups of G with register
// double buffering -- the loads of group g+1 (and of the next chunk's first
// group, across the v-phase) are in flight while group g is computed.
template <class T>
struct PassAcc {
  T cost, prev, dual, dx, mx;
  bool bad;
};

// The elementwise update of one column slice (R rows) and its reductions
// (fused.hpp:249-284).  c = column index within the 16-column staging chunk.
template <class T, int MODE, bool DUAL, bool DX, bool MASK>
__device__ __forceinline__ void compute_col(const PassArgs<T>& a, const T (&x)[16 / sizeof(T)],
                                            const T (&cc)[16 / sizeof(T)], T vj, int64_t col,
                                            int c, int64_t row0, int nvalid,
                                            const T (&ph)[16 / sizeof(T)],
                                            T (&u)[16 / sizeof(T)], PassAcc<T>& acc, T* wbuf,
                                            int lane) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  constexpr bool RC = MODE != kSkip;
  const bool live = !MASK || nvalid > 0;
  T xp[R], st[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    T e = T(0), tv;
    if (RC) {
      e = a.rho * cc[t];
      if (MODE == kPlain1)
        tv = ((x[t] - e) + ph[t]) + vj;
      else
        tv = ((x[t] + ph[t]) + vj) - e;
    } else {
      tv = (x[t] + ph[t]) + vj;
    }
    T p = tv > T(0) ? tv : T(0);
    const bool valid = !MASK || t < nvalid;
    if (MASK && !valid) {
      p = T(0);
      tv = T(0);
    }
    xp[t] = p;
    st[t] = (MODE == kFold) ? p - e : p;
    u[t] += p;
    if (RC) {
      acc.cost = fma(cc[t], p, acc.cost);
      acc.prev = fma(cc[t], x[t], acc.prev);
      if (DUAL) {
        T d = (ph[t] + vj) - e;
        d = d > T(0) ? d : T(0);
        if (MASK && !valid) d = T(0);
        acc.dual = fma(d, d, acc.dual);
      }
    }
    if (DX) {
      const T dd = p - x[t];
      acc.dx = fma(dd, dd, acc.dx);
    }
    const T at = fabs(tv);
    acc.mx = fmax(acc.mx, at);
    acc.bad |= !(at <= max_finite<T>());
  }
  if (live) __stcs(reinterpret_cast<V*>(a.xy + col * a.ld + row0), pack4(st));
  *reinterpret_cast<V*>(wbuf + (c * 32 + (lane ^ (c & 7))) * R) = pack4(xp);
}

// exact accumulation (drotb_internal.hpp kHiScale): split, add, combine
struct HiLo {
  long long hi, lo;
};
__device__ __forceinline__ HiLo to_hilo(double x) {
  const long long hi = __double2ll_rn(x * kHiScale);
  const double rem = x - static_cast<double>(hi) * kHiInv;  // exact
  return HiLo{hi, __double2ll_rn(rem * kLoScale)};
}
__device__ __forceinline__ void hilo_add(HiLo& a, double x) {
  const HiLo h = to_hilo(x);
  a.hi += h.hi;
  a.lo += h.lo;
}
__device__ __forceinline__ double hilo_value(long long hi, long long lo) {
  return static_cast<double>(hi) * kHiInv + static_cast<double>(lo) * kLoInv;
}
__device__ __forceinline__ void red_add_u64(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_hilo(long long* p, const HiLo& h) {
  red_add_u64(p, h.hi);
  red_add_u64(p + 1, h.lo);
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp reduce-scatter of 16 int64 words per lane (butterfly): at levels
// xor 16, 8, 4, 2 each lane sends the half of its words it does not keep and
// adds its partner's other half; xor 1 completes the sum.  Even lane l ends
// with the warp total of word bfly16_word(l).  31 shuffles of 64 bits
// instead of 80 for 16 separate warp sums (~3x faster CTA reductions of the
// tail's exact hi / lo accumulators, scripts/micro/ctasum.cu).
__device__ __forceinline__ long long bfly16(long long (&v)[16], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 4; ++lvl) {
    const int half = 16 >> (lvl + 1);
    const int bit = 16 >> lvl;
    const bool up = (lane & bit) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const long long send = up ? v[i] : v[i + half];
      const long long keep = up ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}
__device__ __forceinline__ int bfly16_word(int lane) {
  return ((lane & 16) ? 8 : 0) | ((lane & 8) ? 4 : 0) | ((lane & 4) ? 2 : 0) |
         ((lane & 2) ? 1 : 0);
}

__device__ __forceinline__ void red_add_fx(long long* p, double v) {
  const long long q = __double2ll_rn(v * kFxScale);
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(q) : "memory");
}
// element i of a fixed-point sum array of length len: fp32 one word at 2^46;
// fp64 a hi word at 2^46 and a lo word (at [len + i]) of the remainder at 2^86
template <class T>
__device__ __forceinline__ void red_fx(long long* base, int64_t i, int64_t len, T v) {
  const double d = static_cast<double>(v);
  const long long hi = __double2ll_rn(d * kFxScale);
  red_add_u64(base + i, hi);
  if (sizeof(T) == 8)
    red_add_u64(base + len + i,
                __double2ll_rn((d - static_cast<double>(hi) * kFxInv) * kFxLoScale));
}

// v-phase: lane (c, b) sums the 64 rows of block b of staged column c in
// row order (fused.hpp:268) and writes the v strip entry -- or, in fixed
// point mode, the warp's column sum joins the column's integer accumulator.
template <class T>
__device__ __forceinline__ void v_phase(const PassArgs<T>& a, const T* wbuf, int64_t j0,
                                        int cnt, int64_t wrow0, int lane) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  constexpr int NB = 32 * R / kVBlockRows;
  constexpr int CH = kChunkCols;
  if (a.fx) {  // one fixed-point red per (column, warp): sum the NB blocks first
    T s = T(0);
    if (lane < CH * NB) {
      const int c = lane % CH, b = lane / CH;
      const int64_t gb = wrow0 / kVBlockRows + b;
      if (c < cnt && gb * kVBlockRows < a.m) {
        const V* col = reinterpret_cast<const V*>(wbuf) + c * 32;
        const int g7 = c & 7;
        constexpr int QB = kVBlockRows / R;
#pragma unroll
        for (int qq = 0; qq < QB; ++qq) {
          T v4[R];
          unpack(col[(b * QB + qq) ^ g7], v4);
#pragma unroll
          for (int t = 0; t < R; ++t) s += v4[t];
        }
      }
    }
#pragma unroll
    for (int o = CH; o < 32; o <<= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane < CH && lane < cnt && wrow0 < a.m) red_fx<T>(a.vfx, j0 + lane, a.n, s);
    return;
  }
  if (lane < CH * NB) {
    const int c = lane % CH, b = lane / CH;
    const int64_t gb = wrow0 / kVBlockRows + b;
    if (c < cnt && gb * kVBlockRows < a.m) {
      const V* col = reinterpret_cast<const V*>(wbuf) + c * 32;
      const int g7 = c & 7;
      constexpr int QB = kVBlockRows / R;  // chunks per 64-row block
      T s = T(0);
#pragma unroll
      for (int qq = 0; qq < QB; ++qq) {
        T v4[R];
        unpack(col[(b * QB + qq) ^ g7], v4);
#pragma unroll
        for (int t = 0; t < R; ++t) s += v4[t];
      }
      st_keep(a.vstrip + gb * a.n + j0 + c, s, a.l2hint);
    }
  }
}

// ---------------------------------------------------------------------------
// K1 (async): the same sweep with a per-lane cp.async ring in shared memory.
// Each lane copies its own 16-B slices of X and C for kAsyncStages-1 column
// groups ahead (LDGSTS, no register cost for data in flight) and consumes
// them in order; completion is per-thread (cp.async.wait_group), so no
// cross-lane synchronisation is needed for the ring.
// ---------------------------------------------------------------------------
#ifndef DROTB_ASYNC_MINB
#define DROTB_ASYNC_MINB 3  // 3 CTAs (12 warps) per SM: caps registers at 170 (r1 tuning)
#endif
#ifndef DROTB_ASYNC_S
#define DROTB_ASYNC_S 4  // ring stages (S-1 groups in flight)
#endif
#ifndef DROTB_ASYNC_G
#define DROTB_ASYNC_G 2  // columns per stage
#endif
constexpr int kAsyncS = DROTB_ASYNC_S;
constexpr int kAsyncG = DROTB_ASYNC_G;
// skip sweeps (no C): the same ring as kAsyncS stages of 2*kAsyncG columns
// of X; DROTB_SKIP_FINE builds 2*kAsyncS stages of kAsyncG columns (more
// columns in flight -- measured equal at 10k^2, r1o)
#ifdef DROTB_SKIP_FINE
constexpr int kSkipS = 2 * kAsyncS, kSkipG = kAsyncG;
#else
constexpr int kSkipS = kAsyncS, kSkipG = 2 * kAsyncG;
#endif

// The streamed X / C reads use plain cp.async.cg: the cache-hinted form
// (an evict_first createpolicy operand, formerly DROTB_L2HINT bits 0 / 2)
// measured slower and mis-compiled in r2 (an uninitialized policy
// descriptor: illegal-instruction traps and wrong loads), so it is gone.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <class T>
constexpr size_t async_smem_bytes() {
  // per warp: ring [S][2][G][32 lanes] x 16 B + staging [16 cols][32 R] x sizeof(T)
  return static_cast<size_t>(kWarpsPerCta) *
         (static_cast<size_t>(kAsyncS) * 2 * kAsyncG * 32 * 16 +
          static_cast<size_t>(kChunkCols) * 32 * 16);
}

// The first S-1 ring stages of pass_tile_async (same slots and addresses):
// they depend on X and C only, so K1 can issue them before it waits for the
// tail that produces phi / varphi (programmatic dependent launch)
template <class T, int MODE>
__device__ __forceinline__ void ring_prime(const PassArgs<T>& a, int64_t c0, int64_t c1,
                                           int64_t row0, bool live,
                                           typename V16<T>::type* ring, int lane) {
  constexpr bool RC = MODE != kSkip;
  constexpr int S = RC ? kAsyncS : kSkipS, G = RC ? kAsyncG : kSkipG;
  constexpr int SLOTS = 2 * kAsyncG * kAsyncS / S;  // 16-B slots per lane and stage
  // the same copies as pass_tile_async's issue()
#pragma unroll
  for (int st = 0; st < S - 1; ++st) {
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int64_t col = c0 + st * G + k;
      if (col < c1 && live) {
        const int64_t off = col * a.ld + row0;
        cp_async16(ring + (st * SLOTS + k) * 32 + lane, a.xy + off);
        if (RC) cp_async16(ring + (st * SLOTS + kAsyncG + k) * 32 + lane, a.cost + off);
      }
    }
    cp_async_commit();
  }
}

// PRIMED: the caller issued the first S-1 stages (ring_prime)
// Returns true when the loop's stop flag (a.stop) is set: read only after
// the first loads of the tile are in flight (its latency overlaps theirs),
// and before anything is written.
template <class T, int MODE, bool DUAL, bool DX, bool MASK, bool PRIMED = false>
__device__ __forceinline__ bool pass_tile_async(const PassArgs<T>& a, int64_t c0, int64_t c1,
                                                int64_t wrow0, int64_t row0, int nvalid,
                                                const T (&ph)[16 / sizeof(T)],
                                                T (&u)[16 / sizeof(T)], PassAcc<T>& acc,
                                                T* wbuf, typename V16<T>::type* ring,
                                                int lane) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  constexpr bool RC = MODE != kSkip;
  // a stage holds 2*kAsyncG 16-B slots per lane: G columns of X and C, or --
  // on skip sweeps, which read no C -- 2G columns of X (same bytes in flight)
  constexpr int S = RC ? kAsyncS : kSkipS, G = RC ? kAsyncG : kSkipG, CH = kChunkCols;
  constexpr int SLOTS = 2 * kAsyncG * kAsyncS / S;  // 16-B slots per lane and stage
  constexpr int NG = CH / G;
  static_assert(NG % S == 0, "stages must divide the groups of a chunk");
  static_assert(SLOTS >= G * (RC ? 2 : 1), "ring slots per stage");
  const bool live = !MASK || nvalid > 0;
  T vb[S][G];
  auto xslot = [&](int st, int k) { return ring + (st * SLOTS + k) * 32 + lane; };
  auto cslot = [&](int st, int k) { return ring + (st * SLOTS + kAsyncG + k) * 32 + lane; };
  auto issue = [&](int st, int64_t jg) {
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int64_t col = jg + k;
      vb[st][k] = T(0);
      if (col < c1) {
        if (live) {
          const int64_t off = col * a.ld + row0;
          cp_async16(xslot(st, k), a.xy + off);
          if (RC) cp_async16(cslot(st, k), a.cost + off);
        }
        vb[st][k] = __ldg(a.varphi + col);
      }
    }
    cp_async_commit();
  };
  if (!PRIMED) {
#pragma unroll
    for (int st = 0; st < S - 1; ++st) issue(st, c0 + st * G);
  } else {  // X / C of the first stages are in flight; varphi only exists now
#pragma unroll
    for (int st = 0; st < S - 1; ++st)
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int64_t col = c0 + st * G + k;
        vb[st][k] = col < c1 ? __ldg(a.varphi + col) : T(0);
      }
  }
  if (a.stop != nullptr && *reinterpret_cast<const volatile int*>(a.stop)) {
    cp_async_wait<0>();
    return true;
  }
  for (int64_t j0 = c0; j0 < c1; j0 += CH) {
#pragma unroll
    for (int gg = 0; gg < NG; ++gg) {
      const int st = gg % S;
      issue((gg + S - 1) % S, j0 + (gg + S - 1) * G);
      cp_async_wait<S - 1>();
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int64_t col = j0 + gg * G + k;
        if (col < c1) {
          T x[R], cc[R];
#pragma unroll
          for (int t = 0; t < R; ++t) x[t] = cc[t] = T(0);
          if (live) {
            unpack(*xslot(st, k), x);
            if (RC) unpack(*cslot(st, k), cc);
          }
          compute_col<T, MODE, DUAL, DX, MASK>(a, x, cc, vb[st][k],
                                               col, gg * G + k, row0, nvalid, ph, u, acc, wbuf,
                                               lane);
        }
      }
    }
    __syncwarp();
    v_phase<T>(a, wbuf, j0, static_cast<int>(imin64(CH, c1 - j0)), wrow0, lane);
    __syncwarp();
  }
  cp_async_wait<0>();
  return false;
}


// One K1 tile (row block bx, column tile by): the body of pass_kernel_async
// after its prologue (one tile per CTA).
// primed: the first ring stages were issued (ring_prime) by the caller.
template <class T, int MODE, bool DUAL, bool DX>
__device__ __forceinline__ void k1_tile(const PassArgs<T>& a, int64_t bx, int64_t by,
                                        int64_t gridx, unsigned char* dyn_smem,
                                        PassAcc<T>* wacc, bool primed, int64_t it_stamp) {
  using V = typename V16<T>::type;
  constexpr int R = 16 / sizeof(T);
  constexpr int ROWS_W = 32 * R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr size_t ring_v = static_cast<size_t>(kAsyncS) * 2 * kAsyncG * 32;  // V per warp
  V* ring = reinterpret_cast<V*>(dyn_smem) + warp * ring_v;
  T* wbuf = reinterpret_cast<T*>(reinterpret_cast<V*>(dyn_smem) + kWarpsPerCta * ring_v) +
            warp * kChunkCols * ROWS_W;
  const int64_t wrow0 = (bx * kWarpsPerCta + warp) * ROWS_W;
  const int64_t row0 = wrow0 + static_cast<int64_t>(lane) * R;
  const int64_t gc = by;
  const int64_t c0 = gc * a.tc;
  const int64_t c1 = imin64(a.n, c0 + a.tc);
  const int64_t nv = a.m - row0;
  const int nvalid = nv <= 0 ? 0 : (nv >= R ? R : static_cast<int>(nv));
  T ph[R], u[R];
  if (nvalid > 0) {
    unpack(ld_keep(reinterpret_cast<const V*>(a.phi + row0)), ph);
  } else {
#pragma unroll
    for (int t = 0; t < R; ++t) ph[t] = T(0);
  }
#pragma unroll
  for (int t = 0; t < R; ++t) u[t] = T(0);
  PassAcc<T> acc{T(0), T(0), T(0), T(0), T(0), false};
  const bool full = __all_sync(0xffffffffu, nvalid == R);
  bool stopped;
  if (primed) {
    if (full)
      stopped = pass_tile_async<T, MODE, DUAL, DX, false, true>(a, c0, c1, wrow0, row0, nvalid,
                                                                ph, u, acc, wbuf, ring, lane);
    else
      stopped = pass_tile_async<T, MODE, DUAL, DX, true, true>(a, c0, c1, wrow0, row0, nvalid,
                                                               ph, u, acc, wbuf, ring, lane);
  } else {
    if (full)
      stopped = pass_tile_async<T, MODE, DUAL, DX, false>(a, c0, c1, wrow0, row0, nvalid, ph, u,
                                                          acc, wbuf, ring, lane);
    else
      stopped = pass_tile_async<T, MODE, DUAL, DX, true>(a, c0, c1, wrow0, row0, nvalid, ph, u,
                                                         acc, wbuf, ring, lane);
  }
  if (stopped) return;  // (every thread reads the same flag)
  if (a.stamps && threadIdx.x == 0) timeline_point(a.stamps, it_stamp, 7, global_ns());
  if (a.fx) {
#pragma unroll
    for (int t = 0; t < R; ++t)
      if (t < nvalid) red_fx<T>(a.ufx, row0 + t, a.ld, u[t]);
  } else if (nvalid > 0) {
    st_keep(reinterpret_cast<V*>(a.ustrip + gc * a.ld + row0), pack4(u), a.l2hint);
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
  if (threadIdx.x == 0) {
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
    if (a.xacc) {  // exact accumulators (the per-CTA sums rounded, then summed exactly)
      red_hilo(a.xacc + 2 * kXaCost, to_hilo(static_cast<double>(out.cost)));
      red_hilo(a.xacc + 2 * kXaPrev, to_hilo(static_cast<double>(out.prev)));
      red_hilo(a.xacc + 2 * kXaDual, to_hilo(static_cast<double>(out.dual)));
      red_hilo(a.xacc + 2 * kXaDx, to_hilo(static_cast<double>(out.dx)));
      atomicMax(reinterpret_cast<unsigned long long*>(a.xacc + kXaMax),
                static_cast<unsigned long long>(
                    __double_as_longlong(static_cast<double>(out.max_abs))));
      if (out.bad) red_add_u64(a.xacc + kXaBad, 1);
    } else {
      st_partial_keep(a.partials + gc * gridx + bx, out);
    }
    if (a.stamps) timeline_point(a.stamps, it_stamp, 1, global_ns());
  }
  // (one tile per CTA: nothing reuses wacc or the ring after this)
}

// ---------------------------------------------------------------------------
// Solve-loop scalar logic shared by the tail kernels and the persistent
// solver kernel (operates on a Book<T>, in global or shared memory)
// ---------------------------------------------------------------------------
// (i % period) == 0 without a 64-bit division in the common period == 1
// (the default check_every / trace_every)
__device__ __forceinline__ bool every(int64_t i, int64_t period) {
  return period == 1 || (i % period) == 0;
}

template <class T>
__device__ __forceinline__ void erg_update(Book<T>* bk, double value) {
  bk->erg_count += 1;
  bk->erg_mean += (value - bk->erg_mean) / static_cast<double>(bk->erg_count);
}

// Pass totals -> FusedPassOutput scalars, step_impl recursions and the
// objective bookkeeping of solve (fused.hpp:346-356; solver.hpp:266,
// 273-277, 418-437).  tot = {cost, prev, dual, dx, max|t|, sum r, |r|^2, |s|^2}.
template <class T>
__device__ void merge_scalars(Book<T>* bk, const TailArgs<T>& t, const T (&tot)[8],
                              int totbad) {
  bk->pass_cost = tot[0];
  bk->pass_prev = tot[1];
  bk->pass_dual = tot[2];
  bk->pass_dx = tot[3];
  bk->pass_max_abs = tot[4];
  bk->pass_bad = totbad;
  if (!t.solver) return;
  const int64_t k = bk->iter;
  bk->folded = t.folded_after;
  if (totbad) {  // solver.hpp:266, 418-422
    bk->failed = 1;
    bk->iterations = k + 1;
    bk->stop = 1;
    return;
  }
  const T beta = tot[5] / static_cast<T>(t.m_global + t.n_global);
  bk->beta = beta;
  bk->coef = T(2) * beta - bk->alpha;
  bk->nr2 = tot[6];
  bk->ns2 = tot[7];
  bk->iterations = k + 1;
  const bool cost_valid = t.reads_cost != 0;
  const bool dual_valid = t.reads_cost && t.want_dual;
  if (!bk->prev_pass_had_cost && cost_valid)
    erg_update(bk, static_cast<double>(tot[1]));
  if (cost_valid) {
    bk->last_cost = static_cast<double>(tot[0]);
    erg_update(bk, bk->last_cost);
  }
  bk->prev_pass_had_cost = cost_valid ? 1 : 0;
  if (dual_valid)
    bk->last_r_dual = sqrt(static_cast<double>(tot[2])) / static_cast<double>(t.rho);
}

// Gate of solve (solver.hpp:439-504) given the O(m+n) sums of this iteration:
// dual value sum_i p_i phi_i/rho + sum_j q_j varphi_j/rho and the rank-two
// fixed-point terms.  Fires the confirm report (graph IF node, or a pause
// when row-sharded) when the stale-dual gate passes.
template <class T>
__device__ void gate_logic(Book<T>* bk, const TailArgs<T>& t, double dual_value, double dphi2,
                           double dphi, double dvarphi2, double dvarphi, double cross,
                           bool write_trace = true) {
  const bool fp = bk->record_trace != 0;
  bk->alpha = bk->alpha - bk->beta;  // solver.hpp:289
  const int64_t k = bk->iter;
  bk->iter = k + 1;
  double fp_residual = __longlong_as_double(0x7ff8000000000000ULL);
  if (fp) {  // rank-two identity (solver.hpp:443-472)
    double fp_sq = static_cast<double>(t.n_global) * dphi2 +
                   static_cast<double>(t.m_global) * dvarphi2 + 2.0 * dphi * dvarphi;
    if (t.reads_cost && t.want_dx) fp_sq += static_cast<double>(bk->pass_dx) + 2.0 * cross;
    fp_residual = sqrt(fmax(fp_sq, 0.0));
  }
  bk->fp_residual = fp_residual;
  const double r_primal = sqrt(static_cast<double>(bk->nr2) + static_cast<double>(bk->ns2));
  const double gap = fabs(bk->last_cost - dual_value);
  const double gap_scale = bk->relative ? 1.0 / (1.0 + fabs(bk->last_cost)) : 1.0;
  bk->r_primal = r_primal;
  bk->dual_value = dual_value;
  bk->gap = gap;
  const bool check = every(k + 1, bk->check_every);
  const bool trace_row = bk->record_trace && every(k + 1, bk->trace_every);
  if (trace_row) {
    if (write_trace && t.trace && bk->trace_rows < bk->trace_cap) {
      TraceRowDev& row = t.trace[bk->trace_rows];
      row.iter = k + 1;
      row.r_primal = r_primal;
      row.r_dual = bk->last_r_dual;
      row.gap = gap;
      row.objective = bk->last_cost;
      row.ergodic_objective = bk->erg_mean;
      row.fixed_point_residual = fp_residual;
    }
    bk->trace_rows += 1;
  }
  const bool fire = check && r_primal * bk->primal_scale <= bk->tol_primal &&
                    bk->last_r_dual <= bk->tol_dual && gap * gap_scale <= bk->tol_gap;
  if (fire) {
    bk->confirm = 1;
    bk->gate_hits += 1;
    if (t.sharded) bk->stop = 2;  // pause: the host runs the collective confirm
  } else if (k + 1 >= bk->max_iters) {
    bk->stop = 1;
  }
  // the confirm report runs only when the gate fires (graph IF node)
  if (t.use_cond && write_trace) cudaGraphSetConditional(t.cond, fire ? 1u : 0u);
}

// report_elem with mu_i = double(phi_i) / rho precomputed once per row
// (the same division, so the slack is bitwise identical)
template <class T>
__device__ __forceinline__ void report_elem_mu(T xv, T cv, double mu_i, double nu_j, T rho,
                                               bool folded, double& obj, double& dsq) {
  const double c = static_cast<double>(cv);
  double x = static_cast<double>(xv);
  if (folded) {
    x += static_cast<double>(rho) * c;
    if (x < 0) x = 0;
  }
  obj += c * x;
  const double slack = mu_i + nu_j - c;
  if (slack > 0) dsq += slack * slack;
}

// report_elem_mu with the two terms accumulated exactly (HiLo): the report
// sums are then independent of the element-to-thread mapping
template <class T>
__device__ __forceinline__ void report_elem_exact(T xv, T cv, double mu_i, double nu_j, T rho,
                                                  bool folded, HiLo (&acc)[2]) {
  const double c = static_cast<double>(cv);
  double x = static_cast<double>(xv);
  if (folded) {
    x += static_cast<double>(rho) * c;
    if (x < 0) x = 0;
  }
  if (x != 0.0) hilo_add(acc[0], c * x);
  const double slack = mu_i + nu_j - c;
  if (slack > 0) hilo_add(acc[1], slack * slack);
}

template <class T>
__device__ __forceinline__ void report_elem(T xv, T cv, T phi_i, double nu_j,
                                            double drho, T rho, bool folded,
                                            double& obj, double& dsq) {
  const double c = static_cast<double>(cv);
  double x = static_cast<double>(xv);
  if (folded) {
    x += static_cast<double>(rho) * c;
    if (x < 0) x = 0;
  }
  obj += c * x;
  const double slack = static_cast<double>(phi_i) / drho + nu_j - c;
  if (slack > 0) dsq += slack * slack;
}

// Exact report of the matched pair and the confirm decision
// (solver.hpp:339-353, 508-519).  obj / dual_sq: the streamed sums.
template <class T>
__device__ void report_decide(Book<T>* bk, double obj, double dual_sq, int always) {
  const double r_primal = sqrt(static_cast<double>(bk->nr2) + static_cast<double>(bk->ns2));
  const double r_dual = sqrt(dual_sq);
  const double gap = fabs(obj - bk->dual_value);
  bk->rep_objective = obj;
  bk->rep_r_primal = r_primal;
  bk->rep_r_dual = r_dual;
  bk->rep_gap = gap;
  if (always) return;
  const double egs = bk->relative ? 1.0 / (1.0 + fabs(obj)) : 1.0;
  if (r_primal * bk->primal_scale <= bk->tol_primal && r_dual <= bk->tol_dual &&
      gap * egs <= bk->tol_gap) {
    bk->converged = 1;
    bk->stop = 1;
  } else {
    bk->confirm = 0;
    bk->stop = bk->iter >= bk->max_iters ? 1 : 0;  // also ends a sharded pause
  }
}


}  // namespace drotb
