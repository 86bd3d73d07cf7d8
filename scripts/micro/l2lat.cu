// Microbenchmark: dependent-load latency from one thread on a B200 --
// L1-bypassing (.cg) pointer chase over buffers of several sizes, with and
// without 147 other CTAs polling one L2 line, plus atomic round trips.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void chase(const unsigned* next, int hops, unsigned* flag, int pollers,
                      unsigned long long* out) {
  if (blockIdx.x == 0) {
    if (threadIdx.x != 0) return;
    unsigned i = 0;
    for (int k = 0; k < 64; ++k) i = __ldcg(next + i);  // warm
    const long long c0 = clock64();
    const unsigned long long t0 = gns();
    for (int k = 0; k < hops; ++k) i = __ldcg(next + i);
    const unsigned long long t1 = gns();
    const long long c1 = clock64();
    out[0] = t1 - t0;
    out[1] = c1 - c0;
    out[2] = i;
    // atomic round trips
    const unsigned long long t2 = gns();
    unsigned v = 0;
    for (int k = 0; k < 256; ++k) v += atomicAdd(flag + 64, 1u + (v & 1));
    out[3] = gns() - t2;
    out[4] = v;
    atomicExch(flag, 1u);
  } else if (pollers && threadIdx.x == 0) {
    while (ld_relaxed(flag) == 0) {
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* flag;
  unsigned long long* out;
  cudaMalloc(&flag, 4096);
  cudaMalloc(&out, 64);
  for (size_t bytes : {64u << 10, 1u << 20, 16u << 20, 64u << 20, 512u << 20}) {
    const size_t n = bytes / 4;
    std::vector<unsigned> h(n);
    // random cyclic permutation over 128-B lines
    const size_t lines = n / 32;
    std::vector<unsigned> perm(lines);
    for (size_t k = 0; k < lines; ++k) perm[k] = static_cast<unsigned>(k);
    unsigned long long s = 88172645463325252ull;
    for (size_t k = lines - 1; k > 0; --k) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      std::swap(perm[k], perm[s % (k + 1)]);
    }
    for (size_t k = 0; k < lines; ++k) h[perm[k] * 32] = perm[(k + 1) % lines] * 32;
    unsigned* d;
    cudaMalloc(&d, bytes);
    cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
    for (int pollers : {0, 1}) {
      cudaMemset(flag, 0, 4096);
      const int hops = 2000;
      chase<<<pollers ? sms : 1, 32>>>(d, hops, flag, pollers, out);
      cudaDeviceSynchronize();
      unsigned long long o[5];
      cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
      printf("buffer %7zu KB, %s: %.0f ns/hop (%.0f cycles), atomic RT %.0f ns\n", bytes >> 10,
             pollers ? "147 CTAs polling one line" : "quiet                    ",
             double(o[0]) / hops, double(o[1]) / hops, double(o[3]) / 256);
    }
    cudaFree(d);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
