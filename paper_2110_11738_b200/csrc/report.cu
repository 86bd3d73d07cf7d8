// report.cu -- residual_report / objective for an arbitrary (plan, cert)
// pair on the device (problem.hpp:155-225).
//
//   row_i   = sum_j x_ij                 (double, ascending j: one thread per row,
//                                          exactly the reference's accumulation)
//   colsum_j = sum_i x_ij                (double, ascending i)
//   obj      = sum_k c_k x_k             (one chain in storage order)
//   dual_sq  = sum_k [mu_i + nu_j - c]_+^2
//   r_primal = sqrt(sum_i (row_i-p_i)^2 + sum_j (colsum_j-q_j)^2)
//   r_dual   = sqrt(dual_sq),  gap = |obj - (sum_i p_i mu_i + sum_j q_j nu_j)|
//
// exact = 1 reproduces every chain in the reference's order (bitwise equal
// report; the storage-order chains are serial, so this is a parity mode);
// exact = 0 sums columns and the scalar chains with fixed parallel trees.
#include <cstdint>

#include "drotb_internal.hpp"

namespace drotb {

namespace {

constexpr int kRrThreads = 256;
constexpr int kRrStage = 2048;

__device__ __forceinline__ double block_sum_d(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < static_cast<int>(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

// row_i - p_i (one thread per row, ascending j as problem.hpp:192-204)
template <class T>
__global__ void __launch_bounds__(kRrThreads)
    rr_rows_kernel(const T* __restrict__ x, const T* __restrict__ p, int64_t m, int64_t n,
                   double* __restrict__ rowdev) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double acc = 0.0;
  int64_t j = 0;
  for (; j + 4 <= n; j += 4) {
    T v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = x[(j + q) * m + i];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += static_cast<double>(v[q]);
  }
  for (; j < n; ++j) acc += static_cast<double>(x[j * m + i]);
  rowdev[i] = acc - static_cast<double>(p[i]);
}

// per column j: colsum_j - q_j (ascending i when EXACT), and -- fast order
// only -- the column's contributions to obj and dual_sq
template <class T, bool EXACT>
__global__ void __launch_bounds__(kRrThreads)
    rr_cols_kernel(const T* __restrict__ x, const T* __restrict__ c, const T* __restrict__ mu,
                   const T* __restrict__ nu, const T* __restrict__ q, int64_t m, int64_t n,
                   double* __restrict__ coldev, double* __restrict__ colobj,
                   double* __restrict__ coldsq) {
  __shared__ double stage[kRrStage];
  __shared__ double sh[32];
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const T* xc = x + j * m;
    const T* cc = c + j * m;
    const double nu_j = static_cast<double>(nu[j]);
    double cs = 0.0, ob = 0.0, ds = 0.0;
    if (EXACT) {
      for (int64_t base = 0; base < m; base += kRrStage) {
        const int cnt = static_cast<int>(m - base < kRrStage ? m - base : kRrStage);
        for (int e = threadIdx.x; e < cnt; e += blockDim.x)
          stage[e] = static_cast<double>(xc[base + e]);
        __syncthreads();
        if (threadIdx.x == 0)
          for (int e = 0; e < cnt; ++e) cs += stage[e];
        __syncthreads();
      }
    } else {
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const double xv = static_cast<double>(xc[i]);
        const double cv = static_cast<double>(cc[i]);
        cs += xv;
        ob += cv * xv;
        const double slack = static_cast<double>(mu[i]) + nu_j - cv;
        if (slack > 0) ds += slack * slack;
      }
      cs = block_sum_d(cs, sh);
      ob = block_sum_d(ob, sh);
      ds = block_sum_d(ds, sh);
    }
    if (threadIdx.x == 0) {
      coldev[j] = cs - static_cast<double>(q[j]);
      if (!EXACT) {
        colobj[j] = ob;
        coldsq[j] = ds;
      }
    }
  }
}

// final reductions in one block.  EXACT: serial chains in the reference's
// orders (obj and dual_sq over storage order, col_sq over j, row_sq over i,
// dual value over i then j), staged through shared memory by the block.
template <class T, bool EXACT>
__global__ void __launch_bounds__(kRrThreads)
    rr_final_kernel(const T* __restrict__ x, const T* __restrict__ c, const T* __restrict__ mu,
                    const T* __restrict__ nu, const T* __restrict__ p, const T* __restrict__ q,
                    int64_t m, int64_t n, const double* __restrict__ rowdev,
                    const double* __restrict__ coldev, const double* __restrict__ colobj,
                    const double* __restrict__ coldsq, double* __restrict__ out /* 4 */) {
  __shared__ double st0[kRrStage], st1[kRrStage];
  __shared__ double sh[32];
  double obj = 0.0, dsq = 0.0, csq = 0.0, rsq = 0.0, dv = 0.0;
  const int tid = threadIdx.x;
  if (EXACT) {
    const int64_t mn = m * n;
    for (int64_t base = 0; base < mn; base += kRrStage) {
      const int cnt = static_cast<int>(mn - base < kRrStage ? mn - base : kRrStage);
      for (int e = tid; e < cnt; e += blockDim.x) {
        const int64_t k = base + e;
        const int64_t j = k / m, i = k - j * m;
        const double xv = static_cast<double>(x[k]);
        const double cv = static_cast<double>(c[k]);
        st0[e] = cv * xv;
        const double slack = static_cast<double>(mu[i]) + static_cast<double>(nu[j]) - cv;
        st1[e] = slack > 0 ? slack * slack : 0.0;  // +0 leaves the chain bitwise unchanged
      }
      __syncthreads();
      if (tid == 0)
        for (int e = 0; e < cnt; ++e) obj += st0[e];
      if (tid == 32)
        for (int e = 0; e < cnt; ++e) dsq += st1[e];
      __syncthreads();
    }
    if (tid == 64) {
      for (int64_t j = 0; j < n; ++j) csq += coldev[j] * coldev[j];
      for (int64_t i = 0; i < m; ++i) rsq += rowdev[i] * rowdev[i];
    }
    if (tid == 96) {
      for (int64_t i = 0; i < m; ++i) dv += static_cast<double>(p[i]) * static_cast<double>(mu[i]);
      for (int64_t j = 0; j < n; ++j) dv += static_cast<double>(q[j]) * static_cast<double>(nu[j]);
    }
    __shared__ double fin[5];
    if (tid == 0) fin[0] = obj;
    if (tid == 32) fin[1] = dsq;
    if (tid == 64) {
      fin[2] = csq;
      fin[3] = rsq;
    }
    if (tid == 96) fin[4] = dv;
    __syncthreads();
    if (tid != 0) return;
    obj = fin[0];
    dsq = fin[1];
    csq = fin[2];
    rsq = fin[3];
    dv = fin[4];
  } else {
    for (int64_t j = tid; j < n; j += blockDim.x) {
      obj += colobj[j];
      dsq += coldsq[j];
      csq += coldev[j] * coldev[j];
      dv += static_cast<double>(q[j]) * static_cast<double>(nu[j]);
    }
    for (int64_t i = tid; i < m; i += blockDim.x) {
      rsq += rowdev[i] * rowdev[i];
      dv += static_cast<double>(p[i]) * static_cast<double>(mu[i]);
    }
    obj = block_sum_d(obj, sh);
    dsq = block_sum_d(dsq, sh);
    csq = block_sum_d(csq, sh);
    rsq = block_sum_d(rsq, sh);
    dv = block_sum_d(dv, sh);
    if (tid != 0) return;
  }
  out[0] = sqrt(rsq + csq);  // r_primal (problem.hpp:220)
  out[1] = sqrt(dsq);        // r_dual
  out[2] = fabs(obj - dv);   // gap
  out[3] = obj;              // objective
}

}  // namespace

template <class T>
void launch_residual_report(const T* x, const T* c, const T* mu, const T* nu, const T* p,
                            const T* q, int64_t m, int64_t n, bool exact, double* scratch,
                            double* out, cudaStream_t st) {
  double* rowdev = scratch;
  double* coldev = rowdev + m;
  double* colobj = coldev + n;
  double* coldsq = colobj + n;
  rr_rows_kernel<T><<<static_cast<unsigned>((m + kRrThreads - 1) / kRrThreads), kRrThreads, 0,
                      st>>>(x, p, m, n, rowdev);
  const unsigned cb = static_cast<unsigned>(n < 148 * 16 ? n : 148 * 16);
  if (exact) {
    rr_cols_kernel<T, true><<<cb, kRrThreads, 0, st>>>(x, c, mu, nu, q, m, n, coldev, colobj,
                                                       coldsq);
    rr_final_kernel<T, true><<<1, kRrThreads, 0, st>>>(x, c, mu, nu, p, q, m, n, rowdev, coldev,
                                                       colobj, coldsq, out);
  } else {
    rr_cols_kernel<T, false><<<cb, kRrThreads, 0, st>>>(x, c, mu, nu, q, m, n, coldev, colobj,
                                                        coldsq);
    rr_final_kernel<T, false><<<1, kRrThreads, 0, st>>>(x, c, mu, nu, p, q, m, n, rowdev,
                                                        coldev, colobj, coldsq, out);
  }
  count_launch(3);
}

template void launch_residual_report<float>(const float*, const float*, const float*,
                                            const float*, const float*, const float*, int64_t,
                                            int64_t, bool, double*, double*, cudaStream_t);
template void launch_residual_report<double>(const double*, const double*, const double*,
                                             const double*, const double*, const double*,
                                             int64_t, int64_t, bool, double*, double*,
                                             cudaStream_t);

}  // namespace drotb
