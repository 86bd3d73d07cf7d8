// Microbenchmark: latency of the tail's scalar decision (gate.cuh
// tail_decide) on one thread, cold (first call after launch) and warm, on a
// shared-memory Book -- separates the decision's own dependent-latency chain
// from instruction-fetch and launch-parameter misses inside the tail.
// With "N f32|f64", the Book is taken from a real session after 20
// iterations of the N x N Gaussian problem (libdrotb200.so).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//          --expt-relaxed-constexpr -I include -o scripts/micro/decide_lat \
//          scripts/micro/decide_lat.cu -Lpaper_2110_11738_b200 -ldrotb200 \
//          -Xlinker -rpath=$PWD/paper_2110_11738_b200
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "../../paper_2110_11738_b200/csrc/gate.cuh"
#include "drotb.h"

using namespace drotb;

template <class T>
__global__ void decide_bench(const Book<T>* g, long long* out) {
  __shared__ Book<T> sb;
  __shared__ DecideIn<T> din;
  if (threadIdx.x != 0) return;
  sb = *g;
  for (int q = 0; q < 8; ++q) din.tot[q] = T(0.25) + T(q);
  din.sum_pa = 0.5;
  din.sum_pr = 0.25;
  din.sum_qb = 0.5;
  din.sum_qs = 0.125;
  din.inv_n_d = 1e-4;
  din.inv_m_d = 1e-4;
  din.mn = 20000;
  din.rho = T(2);
  din.totbad = 0;
  din.folded_after = 1;
  din.reads_cost = 1;
  din.want_dual = 1;
  din.want_dx = 1;
  __syncwarp(1);
  for (int k = 0; k < 6; ++k) {
    const long long c0 = clock64();
    tail_decide<T>(&sb, &din);
    __syncwarp(1);
    const long long c1 = clock64();
    out[k] = c1 - c0;
  }
  out[6] = sb.iter;
}

template <class T>
int run(const Book<T>& b, const char* label) {
  Book<T>* d;
  long long* o;
  cudaMalloc(&d, sizeof(b));
  cudaMalloc(&o, 8 * sizeof(long long));
  cudaMemcpy(d, &b, sizeof(b), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    decide_bench<T><<<1, 32>>>(d, o);
    long long h[8];
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    std::printf("%s rep %d: cycles per call:", label, rep);
    for (int k = 0; k < 6; ++k) std::printf(" %lld", h[k]);
    std::printf("  (iter %lld)\n", h[6]);
  }
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}

template <class T>
int from_session(int64_t nn) {
  drotb_config cfg;
  drotb_config_default(&cfg);
  cfg.tol_primal = -1.0;
  cfg.max_iters = 1 << 30;
  drotb_session* s = nullptr;
  if (drotb_session_create(&s, nn, nn, sizeof(T) == 4 ? 0 : 1, &cfg) != 0) return 2;
  drotb_session_gen_gaussian(s, 5.0, 0, 1);
  drotb_session_init(s, nullptr);
  drotb_session_enqueue(s, 20);
  drotb_session_synchronize(s);
  uint64_t ptrs[4];
  drotb_session_debug_ptrs(s, ptrs);
  Book<T> b;
  cudaMemcpy(&b, reinterpret_cast<const void*>(ptrs[0]), sizeof(b), cudaMemcpyDeviceToHost);
  std::printf("session book: iter %lld check_every %lld trace_every %lld relative %d "
              "record_trace %d alpha %g\n", (long long)b.iter, (long long)b.check_every,
              (long long)b.trace_every, b.relative, b.record_trace, (double)b.alpha);
  drotb_session_destroy(s);
  return run<T>(b, sizeof(T) == 4 ? "session f32" : "session f64");
}

int main(int argc, char** argv) {
  if (argc >= 3) {
    const long long nn = std::atoll(argv[1]);
    return std::strcmp(argv[2], "f64") == 0 ? from_session<double>(nn) : from_session<float>(nn);
  }
  Book<float> b;
  std::memset(&b, 0, sizeof(b));
  b.max_iters = 1 << 30;
  b.check_every = 1;
  b.trace_every = 1;
  b.trace_cap = 1 << 20;
  b.tol_primal = 1e-4;
  b.tol_dual = 1e-4;
  b.tol_gap = 1e-4;
  b.primal_scale = 1.0;
  b.record_trace = 1;
  b.alpha = 0.5f;
  b.sum_p = 1.0;
  b.sum_q = 1.0;
  return run<float>(b, "synthetic");
}
