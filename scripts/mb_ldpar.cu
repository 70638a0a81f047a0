// mb_ldpar.cu — are independent strong (.relaxed.gpu) loads from one thread
// overlapped?  Cycles for N = 1, 2, 4, 9, 16 loads to distinct L2-resident
// lines issued back to back, then consumed; u32 vs u64, strong vs .cg / .ca.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_ldpar scripts/mb_ldpar.cu
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

template <int N, int KIND>
__global__ void k_ld(const unsigned long long* p, int reps, long long* out, unsigned long long* sink) {
  unsigned long long acc = 0;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    unsigned long long v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const unsigned long long* q = p + (size_t)(i * 16 + (r & 7) * 16 * 32) + (acc & 1);
      if (KIND == 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v[i]) : "l"(q) : "memory");
      else if (KIND == 1) {
        unsigned x;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(q) : "memory");
        v[i] = x;
      } else if (KIND == 2) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v[i]) : "l"(q) : "memory");
      else asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v[i]) : "l"(q) : "memory");
    }
#pragma unroll
    for (int i = 0; i < N; ++i) acc += v[i];
  }
  const long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  sink[0] = acc;
}

template <int N, int KIND>
void run(const char* kind, const unsigned long long* p, long long* dout, unsigned long long* sink) {
  k_ld<N, KIND><<<1, 1>>>(p, 10, dout, sink);
  k_ld<N, KIND><<<1, 1>>>(p, 200, dout, sink);
  CK(cudaDeviceSynchronize());
  long long h;
  CK(cudaMemcpy(&h, dout, 8, cudaMemcpyDeviceToHost));
  printf("%-22s N=%2d: %6lld cycles per batch (%5.0f per load)\n", kind, N, h, (double)h / N);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned long long* p;
  long long* dout;
  unsigned long long* sink;
  CK(cudaMalloc(&p, 1 << 20));
  CK(cudaMemset(p, 0, 1 << 20));
  CK(cudaMalloc(&dout, 64));
  CK(cudaMalloc(&sink, 64));
#define RUNK(K, name) run<1, K>(name, p, dout, sink); run<2, K>(name, p, dout, sink); run<4, K>(name, p, dout, sink); \
  run<9, K>(name, p, dout, sink); run<16, K>(name, p, dout, sink);
  RUNK(0, "ld.relaxed.gpu.u64")
  RUNK(1, "ld.relaxed.gpu.u32")
  RUNK(2, "ld.global.cg.u64")
  RUNK(3, "ld.volatile.u64")
  return 0;
}
