// Dev aid: per-iteration overhead of the graph node patterns a fused
// iteration could use on B200 (decides the confirm-report design of the
// single-kernel iteration).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/graph_overhead \
//        scripts/graph_overhead.cu -lcuda
// Every variant is a graph of ITERS iterations of a streaming kernel (grid of
// CTAS CTAs, each reading and writing a 64 KB slab of a 2*CTAS*64 KB buffer,
// last arriving CTA resets the counter and sets the "fired" condition to 0),
// followed per iteration by:
//   0: nothing
//   1: an IF conditional node (condition set to 0 by the kernel)
//   2: an early-exit kernel of 592 CTAs reading the flag
//   3: an early-exit kernel of 1 CTA
//   4: nothing, streaming kernel launched as a programmatic dependent (PDL)
//   5: early-exit kernel of 592 CTAs, both launched with PDL
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

constexpr int kSlab = 64 * 1024 / 16;  // float4 per CTA slab

__global__ void __launch_bounds__(128) streamk(float4* x, unsigned* cnt, int* flag,
                                               unsigned long long cond, int use_cond) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float4* s = x + static_cast<size_t>(blockIdx.x) * kSlab;
  float4* d = x + static_cast<size_t>(gridDim.x + blockIdx.x) * kSlab;
  for (int i = threadIdx.x; i < kSlab; i += 128) {
    float4 v = s[i];
    v.x += 1.f;
    d[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
      *cnt = 0;
      *flag = 0;
      if (use_cond) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(cond), 0);
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void exitk(const int* flag, float* sink) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (*reinterpret_cast<const volatile int*>(flag) == 0) return;
  sink[blockIdx.x] = 1.f;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static void launch(void (*k)(float4*, unsigned*, int*, unsigned long long, int), int grid,
                   bool pdl, cudaStream_t st, float4* x, unsigned* c, int* f,
                   unsigned long long cond, int uc) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, x, c, f, cond, uc);
}

static void launch_exit(int grid, bool pdl, cudaStream_t st, const int* f, float* sink) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, exitk, f, sink);
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? std::atoi(argv[1]) : 3140;
  const int iters = 200;
  float4* x;
  unsigned* cnt;
  int* flag;
  float* sink;
  CK(cudaMalloc(&x, static_cast<size_t>(2) * ctas * kSlab * sizeof(float4)));
  CK(cudaMemset(x, 0, static_cast<size_t>(2) * ctas * kSlab * sizeof(float4)));
  CK(cudaMalloc(&cnt, 64));
  CK(cudaMemset(cnt, 0, 64));
  CK(cudaMalloc(&flag, 64));
  CK(cudaMemset(flag, 0, 64));
  CK(cudaMalloc(&sink, 4096 * 4));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::printf("ctas %d, %.1f MB moved per launch\n", ctas, 2.0 * ctas * 64 * 1024 / 1e6);
  for (int v = 0; v <= 5; ++v) {
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    std::vector<cudaGraphNode_t> deps;
    for (int it = 0; it < iters; ++it) {
      cudaGraphConditionalHandle h = 0;
      if (v == 1) CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
      CK(cudaStreamBeginCaptureToGraph(st, g, deps.empty() ? nullptr : deps.data(), nullptr,
                                       deps.size(), cudaStreamCaptureModeThreadLocal));
      const bool pdl = v == 4 || v == 5;
      launch(streamk, ctas, pdl && it > 0, st, x, cnt, flag, static_cast<unsigned long long>(h),
             v == 1);
      if (v == 2 || v == 5) launch_exit(592, v == 5, st, flag, sink);
      if (v == 3) launch_exit(1, false, st, flag, sink);
      cudaStreamCaptureStatus cs;
      const cudaGraphNode_t* d = nullptr;
      size_t nd = 0;
      CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &d, &nd));
      deps.assign(d, d + nd);
      cudaGraph_t tmp;
      CK(cudaStreamEndCapture(st, &tmp));
      if (v == 1) {
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        CK(cudaGraphAddNode(&cn, g, deps.data(), deps.size(), &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
        launch_exit(592, false, st, flag, sink);
        CK(cudaStreamEndCapture(st, &tmp));
        deps.assign(1, cn);
      }
    }
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(ex, st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0) best = std::min(best, ms);
    }
    std::printf("variant %d: %.2f us / iteration\n", v, best * 1e3f / iters);
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
  }
  CK(cudaGetLastError());
  return 0;
}
