/* drot_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference DROT solver's hot path
 * (/root/reference/proj/core/include/drot/{solver,fused,problem,probgen,rng}.hpp)
 * used as the CPU checker for the B200 product.  It is NOT part of the
 * product: paper_2110_11738_b200/ never links or calls it.  Parity of this
 * restatement with the reference itself is pinned by tests/test_oracle.py
 * against oracle/_ref/libdrotref.so (the unmodified reference compiled here)
 * and against the committed golden vectors under tests/golden/.
 *
 * Build: oracle/Makefile (gcc -O2 -std=c11 -ffp-contract=off: the reference
 * arithmetic is evaluated without FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* drot::Errc ordinals (errors.hpp:24-46). */
enum {
  ORC_ERRC_NEGATIVE_COST = 0,
  ORC_ERRC_MARGINAL_NOT_SIMPLEX = 1,
  ORC_ERRC_EMPTY_DIMENSION = 2,
  ORC_ERRC_NON_FINITE_ENTRY = 3,
  ORC_ERRC_SHAPE_MISMATCH = 4,
  ORC_ERRC_NON_POSITIVE_RHO = 5,
  ORC_ERRC_INVALID_INITIAL_PLAN = 6,
  ORC_ERRC_NON_FINITE_ITERATE = 7,
  ORC_ERRC_DEGENERATE_COST = 10,
  ORC_ERRC_FOLD_STATE_MISMATCH = 12,
};

/* ---- CounterRng: rng.hpp:30-106 (SplitMix64 counter generator) -------- */
static const uint64_t kGolden = 0x9E3779B97F4A7C15ull;

static uint64_t rng_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t orc_derive_key(uint64_t key, uint64_t stream) {
  return rng_mix(key ^ rng_mix(stream + kGolden));
}

typedef struct {
  uint64_t key, counter;
} orc_rng;

static uint64_t rng_next_u64(orc_rng* g) {
  g->counter += kGolden;
  return rng_mix(g->key + g->counter);
}

static double rng_next_unit(orc_rng* g) {
  return (double)(rng_next_u64(g) >> 11) * 0x1.0p-53;
}

static double rng_next_unit_open(orc_rng* g) {
  return ((double)(rng_next_u64(g) >> 11) + 0.5) * 0x1.0p-53;
}

/* Marsaglia polar method, rng.hpp:66-78. */
static void rng_gaussian_pair(orc_rng* g, double* z0, double* z1) {
  for (;;) {
    const double a = 2.0 * rng_next_unit(g) - 1.0;
    const double b = 2.0 * rng_next_unit(g) - 1.0;
    const double s = a * a + b * b;
    if (s > 0.0 && s < 1.0) {
      const double r = sqrt(-2.0 * log(s) / s);
      *z0 = a * r;
      *z1 = b * r;
      return;
    }
  }
}

void orc_rng_u64(uint64_t key, int64_t count, uint64_t* out) {
  orc_rng g = {key, 0};
  for (int64_t k = 0; k < count; ++k) out[k] = rng_next_u64(&g);
}

/* drot_tests::random_matrix / Fixture draws (tests/support/oracles.hpp:128-135):
 * lo + (hi - lo) * next_unit() in storage order. */
void orc_random_unit(uint64_t seed, int64_t count, double lo, double hi,
                     double* out) {
  orc_rng g = {seed, 0};
  for (int64_t k = 0; k < count; ++k) out[k] = lo + (hi - lo) * rng_next_unit(&g);
}

/* ---- gen_gaussian_problem: probgen.hpp:131-170 ------------------------- */
typedef struct {
  double mean[2];
  double factor[4];
} orc_gauss2;

static orc_gauss2 sample_params(uint64_t base, uint64_t mean_stream,
                                uint64_t factor_stream, double shift,
                                double scale) {
  orc_gauss2 g;
  orc_rng mr = {orc_derive_key(base, mean_stream), 0};
  double z0, z1;
  rng_gaussian_pair(&mr, &z0, &z1);
  g.mean[0] = shift + scale * z0;
  g.mean[1] = shift + scale * z1;
  orc_rng fr = {orc_derive_key(base, factor_stream), 0};
  for (int k = 0; k < 4; ++k) g.factor[k] = rng_next_unit(&fr);
  return g;
}

static void sample_points(uint64_t base, const orc_gauss2* g, int64_t count,
                          uint64_t stream0, double* pts /* 2 x count */) {
  for (int64_t i = 0; i < count; ++i) {
    orc_rng r = {orc_derive_key(base, stream0 + (uint64_t)i), 0};
    double z0, z1;
    rng_gaussian_pair(&r, &z0, &z1);
    pts[2 * i + 0] = g->mean[0] + g->factor[0] * z0 + g->factor[2] * z1;
    pts[2 * i + 1] = g->mean[1] + g->factor[1] * z0 + g->factor[3] * z1;
  }
}

int orc_gen_gaussian(int64_t m, int64_t n, double sigma_t, uint64_t seed,
                     int32_t dirichlet, double* C, double* p, double* q) {
  if (m == 0 || n == 0) return 1 + ORC_ERRC_EMPTY_DIMENSION;
  const orc_gauss2 src = sample_params(seed, 0, 1, 0.0, 1.0);
  const orc_gauss2 tgt = sample_params(seed, 2, 3, 5.0, sigma_t);
  double* xs = (double*)malloc(sizeof(double) * 2 * (size_t)m);
  double* xt = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  sample_points(seed, &src, m, 100, xs);
  sample_points(seed, &tgt, n, 100 + (uint64_t)m, xt);
  double cmax = 0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0;
      for (int k = 0; k < 2; ++k) {
        const double d = xs[2 * i + k] - xt[2 * j + k];
        acc += d * d;
      }
      C[j * m + i] = acc;
      const double ab = fabs(acc);
      if (cmax < ab) cmax = ab;
    }
  free(xs);
  free(xt);
  if (!(cmax > 0)) return 1 + ORC_ERRC_DEGENERATE_COST;
  for (int64_t k = 0; k < m * n; ++k) C[k] /= cmax;
  if (dirichlet) {
    /* dirichlet_uniform: probgen.hpp:115-127 */
    for (int pass = 0; pass < 2; ++pass) {
      double* w = pass == 0 ? p : q;
      const int64_t cnt = pass == 0 ? m : n;
      orc_rng r = {orc_derive_key(seed, pass == 0 ? 4 : 5), 0};
      double total = 0;
      for (int64_t k = 0; k < cnt; ++k) {
        w[k] = -log(rng_next_unit_open(&r));
        total += w[k];
      }
      for (int64_t k = 0; k < cnt; ++k) w[k] /= total;
    }
  } else {
    for (int64_t i = 0; i < m; ++i) p[i] = 1.0 / (double)m;
    for (int64_t j = 0; j < n; ++j) q[j] = 1.0 / (double)n;
  }
  return 0;
}

/* drot_tests::random_simplex (tests/support/oracles.hpp:137-147). */
void orc_random_simplex(int64_t n, uint64_t seed, double* out) {
  orc_rng g = {seed, 0};
  double total = 0;
  for (int64_t k = 0; k < n; ++k) {
    out[k] = 0.05 + rng_next_unit(&g);
    total += out[k];
  }
  for (int64_t k = 0; k < n; ++k) out[k] /= total;
}

/* ---- solver restatement, instantiated for float and double ------------- */
#define OT float
#define OSFX f32
#include "drot_oracle_impl.h"
#undef OT
#undef OSFX

#define OT double
#define OSFX f64
#include "drot_oracle_impl.h"
#undef OT
#undef OSFX
