// mb_multi.cu — is the ~100-cycle spacing of warp-wide strong loads per warp
// or per SM?  9 x 256-byte warp loads (lane = row, 8 B each, distinct lines,
// L2-resident), issued by one warp back to back vs. by 9 warps one each
// (released together by a barrier); cycles from the release to all data used.
//   m0  1 warp, 9 loads                 m1  9 warps, 1 load each
//   m2  1 warp, 9 weak ld.global.cg     m3  3 warps, 3 loads each
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_multi scripts/mb_multi.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ldcg(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int M>
__global__ void __launch_bounds__(288, 1) k_multi(const unsigned long long* w, int reps, long long* out,
                                                   unsigned long long* sink) {
  __shared__ unsigned long long acc[9][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long tot = 0;
  unsigned long long s = 0;
  for (int r = 0; r < reps; ++r) {
    const unsigned long long* base = w + (size_t)(r & 15) * 9 * 32 * 2;  // rotate over 16 sets
    __syncthreads();
    const long long t0 = clock64();
    if (M == 0 || M == 2) {
      if (warp == 0) {
        unsigned long long v[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) v[t] = M == 0 ? ldr(base + t * 64 + lane) : ldcg(base + t * 64 + lane);
#pragma unroll
        for (int t = 0; t < 9; ++t) acc[t][lane] = v[t];
      }
    } else if (M == 1) {
      if (warp < 9) acc[warp][lane] = ldr(base + warp * 64 + lane);
    } else {
      if (warp < 3) {
        unsigned long long v[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) v[t] = ldr(base + (warp * 3 + t) * 64 + lane);
#pragma unroll
        for (int t = 0; t < 3; ++t) acc[warp * 3 + t][lane] = v[t];
      }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (warp == 0) {
      unsigned long long x = 0;
      for (int t = 0; t < 9; ++t) x += acc[t][lane];
      s += x;
    }
    if (r > 0) tot += t1 - t0;
  }
  if (threadIdx.x == 0) out[M] = tot / (reps - 1);
  sink[threadIdx.x] = s;
}

template <int M>
void run(const char* name, const unsigned long long* w, long long* dout, unsigned long long* sink) {
  k_multi<M><<<1, 288>>>(w, 100, dout, sink);
  CK(cudaDeviceSynchronize());
  long long h[8];
  CK(cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost));
  printf("%-34s %6lld cycles release -> all 9 x 256 B loaded\n", name, h[M]);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned long long *w, *sink;
  long long* dout;
  CK(cudaMalloc(&w, 16 * 9 * 64 * 8 * 2));
  CK(cudaMemset(w, 1, 16 * 9 * 64 * 8 * 2));
  CK(cudaMalloc(&dout, 64));
  CK(cudaMalloc(&sink, 288 * 8));
  run<0>("m0 1 warp x 9 strong loads", w, dout, sink);
  run<1>("m1 9 warps x 1 strong load", w, dout, sink);
  run<2>("m2 1 warp x 9 ld.global.cg", w, dout, sink);
  run<3>("m3 3 warps x 3 strong loads", w, dout, sink);
  return 0;
}
