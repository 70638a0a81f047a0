// mb_hop.cu — cross-CTA signalling and broadcast-ingress microbenchmarks on
// B200 (design inputs for the tensor-core persistent decoder):
//   A. one-way hop latency, CTA 0 <-> CTA 1 ping-pong:
//      a0 flag only (st.release / ld.acquire)
//      a1 flag only (red.release.add / ld.acquire)
//      a2 8 KB by 128 threads + bar + red.release, reader ld.acquire + bulk copy
//      a3 8 KB + flag, reader: every thread ld.relaxed its 64 B after the flag
//      a4 LL: 16-byte words {d0, epoch, d1, epoch}, reader polls the data itself
//   B. cluster of 2: DSMEM ping-pong with remote mbarrier arrive (8 KB pushed)
//   C. broadcast ingress: G CTAs each bulk-copy the SAME 80 KB (10 x 8 KB chunks)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_hop scripts/mb_hop.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
namespace cg = cooperative_groups;

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
__device__ __forceinline__ void minit(uint64_t* bar, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(128, 1) k_hop(int variant, unsigned char* buf0, unsigned char* buf1, unsigned* ctr,
                                                int iters, long long* out) {
  const int tid = threadIdx.x, me = blockIdx.x;
  if (me > 1) return;
  unsigned char* s = dsm;
  uint64_t* bar = (uint64_t*)(dsm + 8192);
  if (tid == 0) {
    minit(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned char* mine = me == 0 ? buf0 : buf1;
  unsigned char* theirs = me == 0 ? buf1 : buf0;
  unsigned* myc = ctr + me * 32;
  unsigned* thc = ctr + (1 - me) * 32;
  uint32_t ph = 0;
  volatile int sink = 0;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    for (int half = 0; half < 2; ++half) {
      const bool write = (half == 0) == (me == 0);
      if (write) {
        if (variant == 0) {
          __syncthreads();
          if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(myc), "r"((unsigned)it) : "memory");
        } else if (variant == 1) {
          __syncthreads();
          if (tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(myc) : "memory");
        } else if (variant == 2 || variant == 3) {
          int4 v = make_int4(it, tid, half, me);
          int4* d = (int4*)mine;
          for (int i = tid; i < 512; i += 128) d[i] = v;
          if (variant == 2) asm volatile("fence.proxy.async.global;" ::: "memory");
          __syncthreads();
          if (tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(myc) : "memory");
        } else {  // LL: 8-byte {data, epoch} pairs, 512 x 16 B
          int4* d = (int4*)mine;
          for (int i = tid; i < 512; i += 128) {
            int4 v = make_int4(tid, it, i, it);
            asm volatile("st.relaxed.gpu.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(d + i), "r"(v.x), "r"(v.y), "r"(v.z),
                         "r"(v.w)
                         : "memory");
          }
        }
      } else {
        if (variant <= 1) {
          if (tid == 0)
            while (ld_acq(thc) < (unsigned)it) {
            }
          __syncthreads();
        } else if (variant == 2) {
          if (tid == 0) {
            while (ld_acq(thc) < (unsigned)it) {
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(8192) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(s)),
                "l"(theirs), "r"(8192), "r"(su(bar))
                : "memory");
            mwait(bar, ph);
          }
          ph ^= 1;
          __syncthreads();
        } else if (variant == 3) {
          if (tid == 0)
            while (ld_acq(thc) < (unsigned)it) {
            }
          __syncthreads();
          const int4* d = (const int4*)theirs;
          int acc = 0;
          for (int i = tid; i < 512; i += 128) {
            int4 v = __ldcg(d + i);
            acc += v.x;
          }
          sink = acc;
          __syncthreads();
        } else {
          const int4* d = (const int4*)theirs;
          for (int i = tid; i < 512; i += 128) {
            int4 v;
            do {
              asm volatile("ld.relaxed.gpu.global.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                           : "l"(d + i)
                           : "memory");
            } while (v.y != it || v.w != it);
          }
          __syncthreads();
        }
      }
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[me] = t1 - t0;
}

// B: cluster of 2, DSMEM push of 8 KB + remote mbarrier arrive (release.cluster)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_dsmem(int bytes, int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  const unsigned me = cl.block_rank();
  unsigned char* s = dsm;  // receive buffer
  uint64_t* bar = (uint64_t*)(dsm + 16384);
  if (tid == 0) {
    minit(bar, 128);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  unsigned char* rs = cl.map_shared_rank(s, me ^ 1);
  uint64_t* rbar = cl.map_shared_rank(bar, me ^ 1);
  uint32_t rbar_addr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar_addr) : "r"(su(bar)), "r"(me ^ 1));
  (void)rbar;
  uint32_t ph = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int half = 0; half < 2; ++half) {
      const bool write = (half == 0) == (me == 0);
      if (write) {
        int4 v = make_int4(it, tid, half, me);
        for (int i = tid; i < bytes / 16; i += 128) ((int4*)rs)[i] = v;
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar_addr) : "memory");
      } else {
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                su(bar)),
            "r"(ph)
            : "memory");
        ph ^= 1;
      }
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[me] = t1 - t0;
}

// C: every CTA bulk-copies the same nch x 8 KB region into smem, reps times
__global__ void __launch_bounds__(128, 1) k_ingress(const unsigned char* src, int nch, int reps, long long* out) {
  uint64_t* bar = (uint64_t*)(dsm + 10 * 8192);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 10; ++i) minit(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  long long t0 = clock64();
  if (tid == 0) {
    for (int r = 0; r < reps; ++r) {
      for (int c = 0; c < nch; ++c) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[c])), "r"(8192) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su(dsm + c * 8192)),
                     "l"(src + (size_t)c * 8192), "r"(8192), "r"(su(&bar[c]))
                     : "memory");
      }
      for (int c = 0; c < nch; ++c) mwait(&bar[c], r & 1);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d clock %d MHz\n", nsm, clk / 1000);
  unsigned char *b0, *b1;
  unsigned* ctr;
  long long* dh;
  CK(cudaMalloc(&b0, 8192));
  CK(cudaMalloc(&b1, 8192));
  CK(cudaMalloc(&ctr, 256 * 4));
  CK(cudaMalloc(&dh, 256 * 8));
  CK(cudaFuncSetAttribute(k_hop, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 + 64));
  const char* nm[] = {"flag st.release", "flag red.release", "8KB + flag, bulk copy", "8KB + flag, ld.cg",
                      "8KB LL (data polled)"};
  for (int v = 0; v < 5; ++v) {
    const int iters = 2000;
    CK(cudaMemset(ctr, 0, 256 * 4));
    CK(cudaMemset(b0, 0, 8192));
    CK(cudaMemset(b1, 0, 8192));
    k_hop<<<2, 128, 8192 + 64>>>(v, b0, b1, ctr, iters, dh);
    CK(cudaDeviceSynchronize());
    long long h[2];
    CK(cudaMemcpy(h, dh, 16, cudaMemcpyDeviceToHost));
    printf("A%d %-24s: %.0f cycles per one-way hop\n", v, nm[v], (double)h[0] / (2 * iters));
  }
  CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 64));
  for (int bytes : {16, 2048, 8192, 16384}) {
    const int iters = 2000;
    k_dsmem<<<2, 128, 16384 + 64>>>(bytes, iters, dh);
    CK(cudaDeviceSynchronize());
    long long h[2];
    CK(cudaMemcpy(h, dh, 16, cudaMemcpyDeviceToHost));
    printf("B  DSMEM push %5d B + remote arrive: %.0f cycles per one-way hop\n", bytes, (double)h[0] / (2 * iters));
  }
  unsigned char* src;
  CK(cudaMalloc(&src, 10 * 8192));
  CK(cudaMemset(src, 1, 10 * 8192));
  CK(cudaFuncSetAttribute(k_ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 10 * 8192 + 128));
  for (int G : {1, 9, 20, 40, 74, 148}) {
    const int reps = 50;
    k_ingress<<<G, 128, 10 * 8192 + 128>>>(src, 10, 2, dh);
    k_ingress<<<G, 128, 10 * 8192 + 128>>>(src, 10, reps, dh);
    CK(cudaDeviceSynchronize());
    std::vector<long long> h(G);
    CK(cudaMemcpy(h.data(), dh, G * 8, cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (auto x : h) mx = x > mx ? x : mx;
    printf("C  broadcast ingress 80 KB, G=%3d CTAs: %.0f cycles per 80 KB (%.1f B/cycle/SM)\n", G,
           (double)mx / reps, 81920.0 * reps / mx);
  }
  return 0;
}
