// microbench2.cu — L2 -> SM streaming characteristics on B200:
//  bulk-copy (TMA 1-D) ring with varying chunk size / slots, consumer does nothing,
//  and plain LDG.128 streaming with N warps x U loads in flight.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
extern __shared__ __align__(128) unsigned char dsm[];

__global__ void k_bulk(const char* src, int nchunks, int chunk, int ns, int shared, size_t span, float* sink) {
  uint64_t* full = (uint64_t*)dsm;
  uint64_t* empty = full + 16;
  char* ring = (char*)(dsm + 256);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  float acc = 0;
  if (tid == 32) {
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % ns;
      if (c >= ns) asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}" ::"r"(su(&empty[s])), "r"(((c / ns) - 1) & 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(chunk));
      const char* p = src + ((shared ? (size_t)c * chunk : ((size_t)blockIdx.x * nchunks + c) * chunk) % span);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(ring + (size_t)s * chunk)), "l"(p), "r"(chunk), "r"(su(&full[s])) : "memory");
    }
  } else if (tid == 0) {
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % ns;
      asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}" ::"r"(su(&full[s])), "r"((c / ns) & 1));
      acc += *(float*)(ring + (size_t)s * chunk);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])));
    }
  }
  if (acc == 1234.f) sink[0] = acc;
}

// every warp streams its own contiguous region with U independent LDG.128 in flight per lane
template <int U>
__global__ void k_ldg(const float4* src, int iters, int shared, size_t span4, float* sink) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  size_t base = shared ? 0 : ((size_t)blockIdx.x * nw + w) * (size_t)iters * U * 32;
  for (int it = 0; it < iters; ++it) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(src + (base + ((size_t)it * U + u) * 32 + lane) % span4);
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
  }
  if (acc.x == 1234.f) sink[0] = acc.y;
}

int main() {
  size_t span = (size_t)64 << 20;  // 64 MB: L2 resident
  char* src; float* sink;
  CK(cudaMalloc(&src, span)); CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(src, 0, span));
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int chunk : {2048, 8192, 32768}) for (int ns : {2, 4, 8, 16}) {
    if ((size_t)chunk * ns > 190 * 1024) continue;
    for (int shared : {1, 0}) {
      int nchunks = (int)(((size_t)16 << 20) / chunk / 16);  // 1 MB per CTA
      size_t smem = 256 + (size_t)chunk * ns;
      k_bulk<<<148, 64, smem>>>(src, nchunks, chunk, ns, shared, span, sink);
      cudaEventRecord(a);
      k_bulk<<<148, 64, smem>>>(src, nchunks, chunk, ns, shared, span, sink);
      cudaEventRecord(b); CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, a, b);
      double bytes = 148.0 * nchunks * chunk;
      printf("bulk chunk=%5d ns=%2d %s: %.3f us/chunk, per-SM %.1f GB/s, aggregate %.0f GB/s\n", chunk, ns,
             shared ? "shared  " : "distinct", 1000.0 * ms / nchunks, bytes / 148 / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9);
    }
  }
  for (int warps : {4, 8, 16}) for (int shared : {1, 0}) {
    int iters = 64;
    k_ldg<8><<<148, warps * 32>>>((const float4*)src, iters, shared, span / 16, sink);
    cudaEventRecord(a);
    k_ldg<8><<<148, warps * 32>>>((const float4*)src, iters, shared, span / 16, sink);
    cudaEventRecord(b); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = 148.0 * warps * 32 * 16 * 8.0 * iters;
    printf("ldg warps=%2d U=8 %s: per-SM %.1f GB/s, aggregate %.0f GB/s (%.2f us)\n", warps, shared ? "shared  " : "distinct",
           bytes / 148 / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9, ms * 1000);
  }
  return 0;
}
