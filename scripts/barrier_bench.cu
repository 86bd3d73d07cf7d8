// Dev aid: cost of a grid-wide barrier among co-resident CTAs on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier_bench scripts/barrier_bench.cu
// Variants: (0) atomicAdd + volatile spin with __nanosleep, (1) same without
// sleep, (2) cooperative_groups grid.sync(), (3) ld.acquire spin on a
// per-generation flag with red.release arrive.
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_v0(unsigned* bar, unsigned nb, int sleep) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nb - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      if (sleep)
        while (*gen == g) __nanosleep(20);
      else
        while (*gen == g) {
        }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// arrive with one atomic on a counter that never resets: the target of
// barrier number k is k * nb
__device__ __forceinline__ void bar_v3(unsigned* cnt, unsigned nb, unsigned& k) {
  __syncthreads();
  ++k;
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    const unsigned target = k * nb;
    while (static_cast<int>(ld_acquire(cnt) - target) < 0) {
    }
  }
  __syncthreads();
}

__global__ void kbar(unsigned* bar, int iters, int variant) {
  unsigned k = 0;
  for (int i = 0; i < iters; ++i) {
    if (variant == 0) bar_v0(bar, gridDim.x, 1);
    else if (variant == 1) bar_v0(bar, gridDim.x, 0);
    else if (variant == 2) cg::this_grid().sync();
    else bar_v3(bar + 4, gridDim.x, k);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  cudaMalloc(&bar, 64);
  const int iters = 2000;
  for (int per = 1; per <= 4; per *= 2) {
    for (int v = 0; v < 4; ++v) {
      cudaMemset(bar, 0, 64);
      const int grid = sms * per;
      void* args[] = {&bar, (void*)&iters, &v};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaLaunchCooperativeKernel((void*)kbar, grid, 128, args, 0, 0);  // warm
      cudaMemset(bar, 0, 64);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)kbar, grid, 128, args, 0, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %4d variant %d: %.3f us per barrier (%s)\n", grid, v, ms * 1e3 / iters,
             cudaGetErrorString(err));
    }
  }
  return 0;
}
