// Microbenchmark: CTA-wide exact sums of 16 int64 words per thread (the
// tail's hi / lo accumulators) over 448 threads -- warp shuffles (64-bit,
// 5 levels), redux.sync on three 22-bit chunks, and a shared-memory
// transpose.  Prints cycles per reduction and checks the three agree.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -o scripts/micro/ctasum scripts/micro/ctasum.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 448, NW = 16, NWARP = NT / 32;

__device__ __forceinline__ long long shfl_sum(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long redux_sum(long long v) {
  const unsigned c0 = static_cast<unsigned>(v) & 0x3FFFFFu;
  const unsigned c1 = static_cast<unsigned>(v >> 22) & 0x3FFFFFu;
  const int c2 = static_cast<int>(v >> 44);
  const unsigned s0 = __reduce_add_sync(0xffffffffu, c0);
  const unsigned s1 = __reduce_add_sync(0xffffffffu, c1);
  const int s2 = __reduce_add_sync(0xffffffffu, c2);
  return (static_cast<long long>(s2) << 44) + (static_cast<long long>(s1) << 22) +
         static_cast<long long>(s0);
}

// butterfly reduce-scatter over the warp: NW = 16 words per lane; after
// level xor 16/8/4/2 each lane holds one word summed over 16 lanes, xor 1
// completes it; lane l ends with word (l >> 1) (bit-reversed order below)
__device__ __forceinline__ long long bfly16(long long (&v)[NW], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 4; ++lvl) {
    const int half = NW >> (lvl + 1);  // pairs this level: 8, 4, 2, 1
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
// which word lane l holds after bfly16: bits of (l >> 1) select upper halves
__device__ __forceinline__ int bfly16_word(int lane) {
  // level 0 (bit 16) keeps the upper 8 words when lane & 16: word index bit 3
  return ((lane & 16) ? 8 : 0) | ((lane & 8) ? 4 : 0) | ((lane & 4) ? 2 : 0) | ((lane & 2) ? 1 : 0);
}

template <int MODE>
__global__ void __launch_bounds__(NT, 1) bench(const long long* in, long long* out, long long* cyc) {
  __shared__ long long sh[8 * NT];
  __shared__ long long part[NW * NWARP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long v[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) v[k] = in[k * NT + tid];
  __syncthreads();
  long long c0 = clock64();
  long long tot = 0;
  for (int rep = 0; rep < 4; ++rep) {
    long long w[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) w[k] = v[k] + rep;
    if (MODE == 3) {
      const long long s = bfly16(w, lane);
      if ((lane & 1) == 0) part[bfly16_word(lane) * NWARP + warp] = s;
      __syncthreads();
      if (tid < NW) {
        long long t2 = 0;
#pragma unroll
        for (int q = 0; q < NWARP; ++q) t2 += part[tid * NWARP + q];
        tot = t2;
      }
    } else if (MODE == 0 || MODE == 1) {
#pragma unroll
      for (int k = 0; k < NW; ++k) w[k] = MODE == 0 ? shfl_sum(w[k]) : redux_sum(w[k]);
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < NW; ++k) part[k * NWARP + warp] = w[k];
      __syncthreads();
      if (tid < NW) {
        long long s = 0;
#pragma unroll
        for (int q = 0; q < NWARP; ++q) s += part[tid * NWARP + q];
        tot = s;
      }
    } else {
      // transpose, 8 words at a time: row = thread; thread t sums word t % 8
      // over the rows t / 8, t / 8 + 56, ...; lanes l, l + 8, l + 16, l + 24
      // hold the same word
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (half) __syncthreads();
#pragma unroll
        for (int k = 0; k < 8; k += 2)
          *reinterpret_cast<longlong2*>(&sh[tid * 8 + k]) = make_longlong2(w[half * 8 + k], w[half * 8 + k + 1]);
        __syncthreads();
        const int word = tid & 7;
        constexpr int RS = NT / 8;  // 56 row groups
        long long s = 0;
#pragma unroll
        for (int r = tid >> 3; r < NT; r += RS) s += sh[r * 8 + word];
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        s += __shfl_xor_sync(0xffffffffu, s, 16);
        if (lane < 8) part[(half * 8 + word) * NWARP + warp] = s;
      }
      __syncthreads();
      if (tid < NW) {
        long long t2 = 0;
#pragma unroll
        for (int q = 0; q < NWARP; ++q) t2 += part[tid * NWARP + q];
        tot = t2;
      }
    }
    __syncthreads();
  }
  long long c1 = clock64();
  if (tid < NW) out[tid] = tot;
  if (tid == 0) *cyc = (c1 - c0) / 4;
}

int main() {
  long long h[NW * NT];
  unsigned long long x = 88172645463325252ull;
  for (auto& e : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    e = static_cast<long long>(x >> 3) - (1ll << 59);
  }
  long long *din, *dout, *dc;
  cudaMalloc(&din, sizeof(h));
  cudaMalloc(&dout, 4 * NW * sizeof(long long));
  cudaMalloc(&dc, 4 * sizeof(long long));
  cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int it = 0; it < 2; ++it) {
    bench<0><<<1, NT>>>(din, dout, dc);
    bench<1><<<1, NT>>>(din, dout + NW, dc + 1);
    bench<2><<<1, NT>>>(din, dout + 2 * NW, dc + 2);
    bench<3><<<1, NT>>>(din, dout + 3 * NW, dc + 3);
  }
  long long o[4 * NW], c[4];
  cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
  cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
  bool ok = true;
  for (int k = 0; k < NW; ++k)
    ok &= o[k] == o[NW + k] && o[k] == o[2 * NW + k] && o[k] == o[3 * NW + k];
  std::printf("cycles per CTA reduction of %d int64 words x %d threads: shfl %lld, redux %lld, "
              "smem %lld, butterfly %lld; agree %d\n", NW, NT, c[0], c[1], c[2], c[3], ok ? 1 : 0);
  return ok ? 0 : 1;
}
