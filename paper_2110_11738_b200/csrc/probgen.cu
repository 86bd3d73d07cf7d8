// probgen.cu -- K7: on-device generation of the synthetic cost matrices,
// bit-identical to the reference's host generators.
//
//   gaussian cost   squared_euclidean_cost + normalize_cost
//                   (probgen.hpp:54-79, as used by gen_gaussian_problem
//                   :131-170): C_ij = (dx*dx + dy*dy) / cmax in double,
//                   cmax = max_ij |C_ij|, then cast to T
//                   (gen_gaussian_problem_as<T>, :172-180).
//   uniform cost    drot_tests::random_matrix (oracles.hpp:128-135):
//                   C[k] = lo + (hi-lo) * CounterRng(seed).next_unit(), k the
//                   column-major storage index (rng.hpp:49-57).
//
// The points themselves (O(m+n) Marsaglia-polar samples, probgen.hpp:102-113)
// are drawn on the host (probgen.cpp); everything O(m*n) runs here.  The
// library is compiled with -fmad=false and double division is IEEE
// round-to-nearest on the device, so every entry equals the host value bit
// for bit.  Needed for config C5 (10^5 x 10^5 fp32 = 40 GB per matrix, which
// a host cannot generate or hold).
//
// Shards: a rank holding rows [row_begin, row_begin+m) of an m_global-row
// problem generates exactly its rows; cmax is the max over ALL m_global x n
// entries (recomputed on every rank from the replicated points: 10^10 fp64
// distance evaluations at 10^5^2, a few ms, no collective needed).
#include <cstdint>

#include "drotb_internal.hpp"

namespace drotb {

namespace {

__device__ __forceinline__ double sqdist(double2 a, double2 b) {
  // squared_euclidean_cost's loop (probgen.hpp:62-66): acc starts at 0
  double acc = 0.0;
  double d = a.x - b.x;
  acc += d * d;
  d = a.y - b.y;
  acc += d * d;
  return acc;
}

constexpr int kGenThreads = 256;
constexpr int kCmaxCols = 2048;  // target points per cmax block
constexpr int kCostCols = 32;    // columns per cost block

// max_ij |C_ij| over all pairs.  Non-negative doubles order like their bit
// patterns, so the grid-wide max is one 64-bit atomicMax (order-free, exact).
__global__ void __launch_bounds__(kGenThreads)
    gaussian_cmax_kernel(const double2* __restrict__ xs, const double2* __restrict__ xt,
                         int64_t m, int64_t n, unsigned long long* cmax_bits) {
  __shared__ double2 sxt[kGenThreads];
  __shared__ double wmax[kGenThreads / 32];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kGenThreads + threadIdx.x;
  const double2 a = i < m ? xs[i] : make_double2(0.0, 0.0);
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * kCmaxCols;
  const int64_t j1 = j0 + kCmaxCols < n ? j0 + kCmaxCols : n;
  double mx = 0.0;
  for (int64_t jb = j0; jb < j1; jb += kGenThreads) {
    __syncthreads();
    if (jb + threadIdx.x < j1) sxt[threadIdx.x] = xt[jb + threadIdx.x];
    __syncthreads();
    const int cnt = static_cast<int>(j1 - jb < kGenThreads ? j1 - jb : kGenThreads);
    if (i < m)
      for (int t = 0; t < cnt; ++t) mx = fmax(mx, fabs(sqdist(a, sxt[t])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kGenThreads / 32; ++w) mx = fmax(mx, wmax[w]);
    atomicMax(cmax_bits, static_cast<unsigned long long>(__double_as_longlong(mx)));
  }
}

// C[j*ld + i] = T(sqdist(xs[i], xt[j]) / cmax) for the local rows; pad rows
// [m, ld) are written as zero.  One thread per row (coalesced stores down
// each column), kCostCols columns per block.
template <class T>
__global__ void __launch_bounds__(kGenThreads)
    gaussian_cost_kernel(const double2* __restrict__ xs_local, const double2* __restrict__ xt,
                         int64_t m, int64_t n, int64_t ld,
                         const unsigned long long* __restrict__ cmax_bits, T* __restrict__ C) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kGenThreads + threadIdx.x;
  if (i >= ld) return;
  const double cmax = __longlong_as_double(static_cast<long long>(*cmax_bits));
  const bool live = i < m;
  const double2 a = live ? xs_local[i] : make_double2(0.0, 0.0);
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * kCostCols;
  const int64_t j1 = j0 + kCostCols < n ? j0 + kCostCols : n;
  for (int64_t j = j0; j < j1; ++j) {
    const double2 b = __ldg(xt + j);
    C[j * ld + i] = live ? static_cast<T>(sqdist(a, b) / cmax) : T(0);
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.hpp:34-38
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// random_matrix: storage index k of the GLOBAL column-major m_global x n
// matrix is k = j*m_global + (row_begin + i); its value is output k+1 of
// CounterRng(seed) (next_u64: mix(key + ctr*golden) after ++ctr).
template <class T>
__global__ void __launch_bounds__(kGenThreads)
    uniform_cost_kernel(uint64_t seed, double lo, double hi, int64_t m, int64_t m_global,
                        int64_t row_begin, int64_t n, int64_t ld, T* __restrict__ C) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kGenThreads + threadIdx.x;
  if (i >= ld) return;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * kCostCols;
  const int64_t j1 = j0 + kCostCols < n ? j0 + kCostCols : n;
  const double span = hi - lo;
  for (int64_t j = j0; j < j1; ++j) {
    T val = T(0);
    if (i < m) {
      const uint64_t k = static_cast<uint64_t>(j * m_global + row_begin + i);
      const uint64_t z = mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull);
      const double unit = static_cast<double>(z >> 11) * 0x1.0p-53;
      val = static_cast<T>(lo + span * unit);
    }
    C[j * ld + i] = val;
  }
}

}  // namespace

void launch_gaussian_cmax(const double* xs, const double* xt, int64_t m, int64_t n,
                          unsigned long long* cmax_bits, cudaStream_t st) {
  cudaMemsetAsync(cmax_bits, 0, sizeof(unsigned long long), st);
  dim3 grid(static_cast<unsigned>((m + kGenThreads - 1) / kGenThreads),
            static_cast<unsigned>((n + kCmaxCols - 1) / kCmaxCols));
  gaussian_cmax_kernel<<<grid, kGenThreads, 0, st>>>(reinterpret_cast<const double2*>(xs),
                                                     reinterpret_cast<const double2*>(xt), m, n,
                                                     cmax_bits);
  count_launch();
}

template <class T>
void launch_gaussian_cost(const double* xs_local, const double* xt, int64_t m, int64_t n,
                          int64_t ld, const unsigned long long* cmax_bits, T* C,
                          cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((ld + kGenThreads - 1) / kGenThreads),
            static_cast<unsigned>((n + kCostCols - 1) / kCostCols));
  gaussian_cost_kernel<T><<<grid, kGenThreads, 0, st>>>(
      reinterpret_cast<const double2*>(xs_local), reinterpret_cast<const double2*>(xt), m, n, ld,
      cmax_bits, C);
  count_launch();
}

template <class T>
void launch_uniform_cost(uint64_t seed, double lo, double hi, int64_t m, int64_t m_global,
                         int64_t row_begin, int64_t n, int64_t ld, T* C, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((ld + kGenThreads - 1) / kGenThreads),
            static_cast<unsigned>((n + kCostCols - 1) / kCostCols));
  uniform_cost_kernel<T><<<grid, kGenThreads, 0, st>>>(seed, lo, hi, m, m_global, row_begin, n,
                                                       ld, C);
  count_launch();
}

template void launch_gaussian_cost<float>(const double*, const double*, int64_t, int64_t,
                                          int64_t, const unsigned long long*, float*,
                                          cudaStream_t);
template void launch_gaussian_cost<double>(const double*, const double*, int64_t, int64_t,
                                           int64_t, const unsigned long long*, double*,
                                           cudaStream_t);
template void launch_uniform_cost<float>(uint64_t, double, double, int64_t, int64_t, int64_t,
                                         int64_t, int64_t, float*, cudaStream_t);
template void launch_uniform_cost<double>(uint64_t, double, double, int64_t, int64_t, int64_t,
                                          int64_t, int64_t, double*, cudaStream_t);

}  // namespace drotb
