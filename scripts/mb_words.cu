// mb_words.cu — latency of the tensor executor's decision hand-off in
// isolation: NW writer CTAs each store 32 tagged 8-byte words (one per row,
// 32 lanes), NR reader CTAs spin (lane = row) until all NW words of their row
// carry the step tag; reader 0 then acks with a tagged word the writers spin
// on.  One iteration = words hop + ack hop.
//   w0  st.relaxed.gpu.u64 words, readers ld.relaxed.gpu.u64, NR = 20
//   w1  as w0 with NR = 1
//   w2  words written with atom.exch (executes at L2)
//   w3  as w0 but the readers poll one word per lane per round (tile by tile)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_words scripts/mb_words.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>

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
__device__ __forceinline__ void str(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int NW = 9;

template <int V>
__global__ void __launch_bounds__(64, 1) k_words(unsigned long long* words, unsigned long long* ack, int nr,
                                                 int iters, long long* out, long long delay) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int me = blockIdx.x;
  const long long t0 = clock64();
  if (me < NW) {  // writer
    for (int it = 1; it <= iters; ++it) {
      if (delay) {  // readers spin this long before the words are written
        const long long d0 = clock64();
        while (clock64() - d0 < delay) {
        }
      }
      const long long tw = clock64();
      if (warp == 0) {
        const unsigned long long w = ((unsigned long long)it << 32) | (unsigned)(me * 32 + lane);
        if (V == 2) atomicExch(&words[me * 32 + lane], w);
        else str(&words[me * 32 + lane], w);
      }
      // wait for the ack of this iteration
      if (threadIdx.x == 0) {
        while ((ldr(ack) >> 32) != (unsigned long long)it) {
        }
        if (me == 0) out[64 + (it & 63)] = clock64() - tw;
      }
      __syncthreads();
    }
  } else if (me < NW + nr) {  // reader
    for (int it = 1; it <= iters; ++it) {
      if (warp == 0) {
        unsigned long long a[NW];
        if (V == 3) {
          for (int t = 0; t < NW; ++t)
            do a[t] = ldr(&words[t * 32 + lane]); while ((a[t] >> 32) < (unsigned long long)it);
        } else {
          for (int t = 0; t < NW; ++t) a[t] = 0;
          bool ok;
          do {
            ok = true;
#pragma unroll
            for (int t = 0; t < NW; ++t)
              a[t] = ldr(&words[t * 32 + lane]);
#pragma unroll
            for (int t = 0; t < NW; ++t) ok = ok && (a[t] >> 32) >= (unsigned long long)it;
          } while (!ok);
        }
        __syncwarp();
        if (me == NW && lane == 0) str(ack, (unsigned long long)it << 32);
      }
      __syncthreads();
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[me] = t1 - t0;
}

template <int V>
void run(const char* name, int nr, unsigned long long* words, unsigned long long* ack, long long* dout,
         long long delay = 0) {
  const int iters = 200;
  CK(cudaMemset(words, 0, NW * 32 * 8));
  CK(cudaMemset(ack, 0, 8));
  k_words<V><<<NW + nr, 64>>>(words, ack, nr, iters, dout, delay);
  CK(cudaDeviceSynchronize());
  long long h[128];
  CK(cudaMemcpy(h, dout, 128 * 8, cudaMemcpyDeviceToHost));
  std::sort(h + 64, h + 128);
  printf("%-48s delay %6lld: write->ack round trip median %6lld cycles\n", name, delay, h[96]);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned long long *words, *ack;
  long long* dout;
  CK(cudaMalloc(&words, NW * 32 * 8));
  CK(cudaMalloc(&ack, 8));
  CK(cudaMalloc(&dout, 128 * 8));
  for (long long d : {0LL, 2000LL, 10000LL, 30000LL}) {
    run<0>("w0 relaxed words, 20 readers", 20, words, ack, dout, d);
    run<0>("w0 relaxed words, 55 readers", 55, words, ack, dout, d);
    run<1>("w1 relaxed words, 1 reader", 1, words, ack, dout, d);
  }
  return 0;
}
