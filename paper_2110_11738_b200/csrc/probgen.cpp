// probgen.cpp -- synthetic instance generation (host), bit-identical to the
// reference generator:
//   CounterRng                 rng.hpp:30-106   (SplitMix64 counter stream)
//   gen_gaussian_problem       probgen.hpp:131-170 (frozen substream layout
//                              probgen.hpp:32-39)
//   gen_gaussian_problem_as<T> probgen.hpp:172-180 (double, normalized, cast)
// plus dyadic-exact simplex marginals, a B200-side input
// fix: the reference's |sum p - 1| <= 1e-12 check (problem.hpp:114) rejects
// plain 1/m marginals in fp32 and at m >= 40000 in fp64.
//
// The cost matrix is computed in parallel over column blocks with
// std::thread; each entry is a pure function of (i, j) so the result does
// not depend on the thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "drotb_host.hpp"

namespace drotb {

template <class F>
void parallel_range(int64_t n, F&& fn) {
  unsigned hc = std::thread::hardware_concurrency();
  const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(hc ? hc : 1, n / 65536 + 1));
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] { fn(n * t / nt, n * (t + 1) / nt); });
  for (auto& x : th) x.join();
}

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

struct Stream {
  uint64_t key, ctr = 0;
  explicit Stream(uint64_t k) : key(k) {}
  uint64_t next() {
    ctr += kGolden;
    return mix64(key + ctr);
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double unit_open() {
    return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53;
  }
  void gauss_pair(double& z0, double& z1) {  // Marsaglia polar, rng.hpp:66-78
    for (;;) {
      const double a = 2.0 * unit() - 1.0;
      const double b = 2.0 * unit() - 1.0;
      const double s = a * a + b * b;
      if (s > 0.0 && s < 1.0) {
        const double r = std::sqrt(-2.0 * std::log(s) / s);
        z0 = a * r;
        z1 = b * r;
        return;
      }
    }
  }
};

inline uint64_t substream_key(uint64_t key, uint64_t stream) {
  return mix64(key ^ mix64(stream + kGolden));
}

struct Cloud {
  double mean[2];
  double f[4];  // column-major 2x2 factor
};

Cloud cloud_params(uint64_t seed, uint64_t mean_stream, uint64_t factor_stream,
                   double shift, double scale) {
  Cloud g;
  Stream ms(substream_key(seed, mean_stream));
  double z0, z1;
  ms.gauss_pair(z0, z1);
  g.mean[0] = shift + scale * z0;
  g.mean[1] = shift + scale * z1;
  Stream fs(substream_key(seed, factor_stream));
  for (double& v : g.f) v = fs.unit();
  return g;
}

void cloud_points(uint64_t seed, const Cloud& g, int64_t count,
                  uint64_t stream0, std::vector<double>& pts) {
  pts.resize(2 * static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) {
    Stream s(substream_key(seed, stream0 + static_cast<uint64_t>(i)));
    double z0, z1;
    s.gauss_pair(z0, z1);
    pts[2 * i + 0] = g.mean[0] + g.f[0] * z0 + g.f[2] * z1;
    pts[2 * i + 1] = g.mean[1] + g.f[1] * z0 + g.f[3] * z1;
  }
}

template <class F>
void parallel_cols(int64_t n, F&& fn) {
  unsigned hc = std::thread::hardware_concurrency();
  const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(hc ? hc : 1, n));
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const int64_t j0 = n * t / nt, j1 = n * (t + 1) / nt;
      fn(j0, j1);
    });
  for (auto& x : th) x.join();
}

inline double sqdist(const double* a, const double* b) {
  double acc = 0;
  for (int k = 0; k < 2; ++k) {
    const double d = a[k] - b[k];
    acc += d * d;
  }
  return acc;
}

}  // namespace

// The m source and n target points (probgen.hpp:150-153), interleaved
// (x, y) per point.  O(m+n): the O(m*n) cost runs on the device (probgen.cu).
int gaussian_points(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                    std::vector<double>& xs, std::vector<double>& xt) {
  if (m <= 0 || n <= 0)
    return set_error(DROTB_ERRC_EMPTY_DIMENSION, "gen_gaussian_problem");
  if (!(sigma_t > 0)) return set_error(DROTB_ERRC_BAD_CONFIG, "sigma_t must be positive");
  const Cloud src = cloud_params(seed, 0, 1, 0.0, 1.0);
  const Cloud tgt = cloud_params(seed, 2, 3, 5.0, sigma_t);
  cloud_points(seed, src, m, 100, xs);
  cloud_points(seed, tgt, n, 100 + static_cast<uint64_t>(m), xt);
  return 0;
}

int gen_gaussian_points(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                        std::vector<double>& xs, std::vector<double>& xt,
                        double* cmax_out) {
  int rc = gaussian_points(m, n, sigma_t, seed, xs, xt);
  if (rc) return rc;
  // cmax = max_ij |C_ij| of the unnormalized cost (probgen.hpp:378-379)
  std::vector<double> colmax(static_cast<size_t>(n), 0.0);
  parallel_cols(n, [&](int64_t j0, int64_t j1) {
    for (int64_t j = j0; j < j1; ++j) {
      double cm = 0;
      for (int64_t i = 0; i < m; ++i)
        cm = std::max(cm, std::abs(sqdist(&xs[2 * i], &xt[2 * j])));
      colmax[j] = cm;
    }
  });
  double cmax = 0;
  for (double v : colmax) cmax = std::max(cmax, v);
  if (!(cmax > 0)) return set_error(DROTB_ERRC_DEGENERATE_COST, "all samples coincide");
  *cmax_out = cmax;
  return 0;
}

// Rows [row_begin, row_end) of the m x n instance (column-major, leading
// dimension row_end - row_begin); the normalization uses the global max.
template <class T>
int gen_gaussian_cost_rows(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                           int64_t row_begin, int64_t row_end, T* C) {
  std::vector<double> xs, xt;
  double cmax = 0;
  int rc = gen_gaussian_points(m, n, sigma_t, seed, xs, xt, &cmax);
  if (rc) return rc;
  const int64_t ml = row_end - row_begin;
  parallel_cols(n, [&](int64_t j0, int64_t j1) {
    for (int64_t j = j0; j < j1; ++j) {
      T* col = C + j * ml;
      for (int64_t i = row_begin; i < row_end; ++i)
        col[i - row_begin] = static_cast<T>(sqdist(&xs[2 * i], &xt[2 * j]) / cmax);
    }
  });
  return 0;
}
template int gen_gaussian_cost_rows<float>(int64_t, int64_t, double, uint64_t, int64_t,
                                           int64_t, float*);
template int gen_gaussian_cost_rows<double>(int64_t, int64_t, double, uint64_t, int64_t,
                                            int64_t, double*);

template <class T>
int gen_gaussian_cost(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                      T* C) {
  return gen_gaussian_cost_rows<T>(m, n, sigma_t, seed, 0, m, C);
}
template int gen_gaussian_cost<float>(int64_t, int64_t, double, uint64_t, float*);
template int gen_gaussian_cost<double>(int64_t, int64_t, double, uint64_t, double*);

void dirichlet_marginal(uint64_t seed, uint64_t stream, int64_t count,
                        double* w) {  // probgen.hpp:115-127
  Stream s(substream_key(seed, stream));
  double total = 0;
  for (int64_t k = 0; k < count; ++k) {
    w[k] = -std::log(s.unit_open());
    total += w[k];
  }
  for (int64_t k = 0; k < count; ++k) w[k] /= total;
}

// drot_tests::random_simplex (oracles.hpp:137-147): 0.05 + next_unit(),
// sequential double total, then w /= total.
void random_simplex(int64_t count, uint64_t seed, double* w) {
  double total = 0;
  for (int64_t k = 0; k < count; ++k) {
    const uint64_t z = mix64(seed + static_cast<uint64_t>(k + 1) * kGolden);
    w[k] = 0.05 + static_cast<double>(z >> 11) * 0x1.0p-53;
    total += w[k];
  }
  for (int64_t k = 0; k < count; ++k) w[k] /= total;
}

template <class T>
int dyadic_marginal(int64_t len, T* out) {
  if (len <= 0) return set_error(DROTB_ERRC_EMPTY_DIMENSION, "dyadic marginal");
  int fl = 0;
  while ((int64_t(1) << (fl + 1)) <= len) ++fl;  // floor(log2 len)
  const int mant = sizeof(T) == 4 ? 23 : 52;
  const int K = std::min(52, mant + fl);
  const uint64_t total = uint64_t(1) << K;
  const uint64_t base = total / static_cast<uint64_t>(len);
  const uint64_t extra = total - base * static_cast<uint64_t>(len);
  const double scale = std::ldexp(1.0, -K);
  for (int64_t k = 0; k < len; ++k) {
    const uint64_t kk = base + (static_cast<uint64_t>(k) < extra ? 1 : 0);
    out[k] = static_cast<T>(static_cast<double>(kk) * scale);
  }
  return 0;
}
template int dyadic_marginal<float>(int64_t, float*);
template int dyadic_marginal<double>(int64_t, double*);

}  // namespace drotb

extern "C" {

int drotb_gen_gaussian(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                       int32_t dirichlet, double* C, double* p, double* q) {
  drotb::clear_error();
  int rc = drotb::gen_gaussian_cost<double>(m, n, sigma_t, seed, C);
  if (rc) return rc;
  if (dirichlet) {
    drotb::dirichlet_marginal(seed, 4, m, p);
    drotb::dirichlet_marginal(seed, 5, n, q);
  } else {
    for (int64_t i = 0; i < m; ++i) p[i] = 1.0 / static_cast<double>(m);
    for (int64_t j = 0; j < n; ++j) q[j] = 1.0 / static_cast<double>(n);
  }
  return 0;
}

int drotb_gen_gaussian_f32(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                           float* C) {
  drotb::clear_error();
  return drotb::gen_gaussian_cost<float>(m, n, sigma_t, seed, C);
}

int drotb_counter_uniform(uint64_t seed, int64_t count, double lo, double hi,
                          double* out) {
  // lo + (hi - lo) * CounterRng(seed).next_unit() for outputs 1..count
  // (rng.hpp:49-57; the reference fixture random_matrix, oracles.hpp:128-135)
  drotb::clear_error();
  if (count < 0) return drotb::set_error(DROTB_ERRC_BAD_CONFIG, "negative count");
  drotb::parallel_range(count, [&](int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k) {
      const uint64_t z = drotb::mix64(seed + static_cast<uint64_t>(k + 1) * 0x9E3779B97F4A7C15ull);
      out[k] = lo + (hi - lo) * (static_cast<double>(z >> 11) * 0x1.0p-53);
    }
  });
  return 0;
}

int drotb_dyadic_marginal_f32(int64_t len, float* out) {
  drotb::clear_error();
  return drotb::dyadic_marginal<float>(len, out);
}
int drotb_dyadic_marginal_f64(int64_t len, double* out) {
  drotb::clear_error();
  return drotb::dyadic_marginal<double>(len, out);
}

}  // extern "C"
