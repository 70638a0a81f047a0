// mb_pub.cu — cost of publishing 16 KB of activations + a counter bump, seen
// from the producer (cycles until the counter bump is issued) and end to end
// (ping-pong between two CTAs, consumer polls then bulk-copies the data).
//   p0  256 threads STG.U16-style 4-byte stores + bar + red.release.gpu (MEMBAR.GPU)
//   p1  same stores + bar + fence.acq_rel.gpu + red.relaxed
//   p2  stage in smem + fence.proxy.async.shared + bar + 2 x 8 KB cp.async.bulk
//       smem->global + commit + wait_group 0 + red.relaxed
//   p3  as p2 with wait_group.read (source reuse only) -- not a visibility
//       guarantee; shows what the write round trip costs
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_pub scripts/mb_pub.cu
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
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
extern __shared__ __align__(1024) unsigned char dsm[];
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mwait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su(bar)), "r"(ph) : "memory");
}

template <int V>
__global__ void __launch_bounds__(256, 1) k_pub(unsigned char* b0, unsigned char* b1, unsigned* ctr, int iters,
                                                long long* out) {
  const int tid = threadIdx.x, me = blockIdx.x;
  if (me > 1) return;
  unsigned char* stage = dsm;                 // 16 KB staging
  unsigned char* rx = dsm + 16384;            // 16 KB receive
  uint64_t* bar = (uint64_t*)(dsm + 32768);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned char* mine = me == 0 ? b0 : b1;
  unsigned char* theirs = me == 0 ? b1 : b0;
  unsigned* myc = ctr + me * 32;
  unsigned* thc = ctr + (1 - me) * 32;
  uint32_t ph = 0;
  long long wsum = 0;
  const long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    for (int half = 0; half < 2; ++half) {
      const bool write = (half == 0) == (me == 0);
      if (write) {
        const long long w0 = clock64();
        if (V <= 1) {
          uint32_t* d = (uint32_t*)mine;
          for (int i = tid; i < 4096; i += 256) d[i] = it + i;
          __syncthreads();
          if (tid == 0) {
            if (V == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(myc) : "memory");
            else {
              asm volatile("fence.acq_rel.gpu;" ::: "memory");
              asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(myc) : "memory");
            }
          }
        } else {
          uint32_t* d = (uint32_t*)stage;
          for (int i = tid; i < 4096; i += 256) d[i] = it + i;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
          if (tid == 0) {
            for (int c = 0; c < 2; ++c)
              asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(mine + c * 8192),
                           "r"(su(stage + c * 8192)), "r"(8192)
                           : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (V == 2) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(myc) : "memory");
          }
        }
        if (tid == 0) wsum += clock64() - w0;
        __syncthreads();
      } else {
        if (tid == 0) {
          while (ld_relaxed(thc) < (unsigned)it) {
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(16384) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           su(rx)),
                       "l"(theirs), "r"(16384), "r"(su(bar))
                       : "memory");
          mwait(bar, ph);
        }
        ph ^= 1;
        __syncthreads();
      }
    }
  }
  const long long t1 = clock64();
  if (tid == 0) {
    out[me * 2] = t1 - t0;
    out[me * 2 + 1] = wsum;
  }
}

template <int V>
void run(const char* name, unsigned char* b0, unsigned char* b1, unsigned* ctr, long long* dout) {
  CK(cudaFuncSetAttribute(k_pub<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 64));
  const int iters = 1000;
  CK(cudaMemset(ctr, 0, 256 * 4));
  k_pub<V><<<2, 256, 32768 + 64>>>(b0, b1, ctr, iters, dout);
  CK(cudaDeviceSynchronize());
  long long h[4];
  CK(cudaMemcpy(h, dout, 32, cudaMemcpyDeviceToHost));
  printf("%-52s one-way hop %6.0f cycles, producer publish %6.0f cycles\n", name, (double)h[0] / (2 * iters),
         (double)h[1] / iters);
}

int main() {
  unsigned char *b0, *b1;
  unsigned* ctr;
  long long* dout;
  CK(cudaMalloc(&b0, 16384));
  CK(cudaMalloc(&b1, 16384));
  CK(cudaMalloc(&ctr, 256 * 4));
  CK(cudaMalloc(&dout, 64));
  run<0>("p0 STG + bar + red.release.gpu", b0, b1, ctr, dout);
  run<1>("p1 STG + bar + fence.acq_rel.gpu + red.relaxed", b0, b1, ctr, dout);
  run<2>("p2 smem + bulk S2G + wait_group 0 + red.relaxed", b0, b1, ctr, dout);
  run<3>("p3 smem + bulk S2G + wait_group.read + red.relaxed", b0, b1, ctr, dout);
  return 0;
}
