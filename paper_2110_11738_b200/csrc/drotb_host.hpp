// drotb_host.hpp -- host-side helpers of libdrotb200.so: the error
// convention of drot::fail (errors.hpp:86-88) mapped onto the C ABI, and the
// host generator entry points.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>
#include <string>
#include <vector>

#include "../../include/drotb.h"

namespace drotb {

// Records "<errc_name>: <what>" (errors.hpp:86-88) and returns 1 + errc.
int set_error(int errc, const std::string& what);
// CUDA / NCCL failures (codes >= DROTB_ERR_CUDA).
int set_cuda_error(int code, const std::string& what);
void clear_error();
const char* last_error_cstr();
const char* errc_name(int errc);

int gaussian_points(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                    std::vector<double>& xs, std::vector<double>& xt);
void random_simplex(int64_t count, uint64_t seed, double* w);
int gen_gaussian_points(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                        std::vector<double>& xs, std::vector<double>& xt,
                        double* cmax_out);
template <class T>
int gen_gaussian_cost(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                      T* C);
template <class T>
int gen_gaussian_cost_rows(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                           int64_t row_begin, int64_t row_end, T* C);
void dirichlet_marginal(uint64_t seed, uint64_t stream, int64_t count,
                        double* w);
template <class T>
int dyadic_marginal(int64_t len, T* out);

}  // namespace drotb

// Error propagation helpers of the host code (C ABI return codes).
#define CUDA_TRY(expr)                                                       \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return ::drotb::set_cuda_error(DROTB_ERR_CUDA + static_cast<int>(e_),  \
                            std::string("cuda: ") + #expr + ": " +           \
                                cudaGetErrorString(e_));                     \
  } while (0)

#define RC_TRY(expr)          \
  do {                        \
    int rc_ = (expr);         \
    if (rc_) return rc_;      \
  } while (0)

