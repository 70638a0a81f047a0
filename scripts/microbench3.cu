// microbench3.cu — per-SM L2->smem streaming: bulk copies issued by many warps
// (one ring per warp) and cp.async (LDGSTS) rings.  148 CTAs, 1 per SM.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
extern __shared__ __align__(128) unsigned char dsm[];

// each warp w: own ring of ns slots x chunk bytes; lane 0 issues, lane 0 consumes
__global__ void k_bulk_mw(const char* src, int nchunks, int chunk, int ns, size_t span, float* sink) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint64_t* full = (uint64_t*)dsm + w * 16;
  char* ring = (char*)(dsm + 16 * 8 * 32) + (size_t)w * ns * chunk;
  if (lane == 0) {
    for (int i = 0; i < ns; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  float acc = 0;
  if (lane == 0) {
    for (int c = 0; c < nchunks + ns; ++c) {
      if (c >= ns) {  // consume c - ns
        const int s = (c - ns) % ns;
        asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}" ::"r"(su(&full[s])), "r"(((c - ns) / ns) & 1));
        acc += *(float*)(ring + (size_t)s * chunk);
      }
      if (c < nchunks) {
        const int s = c % ns;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(chunk));
        const char* p = src + (((size_t)blockIdx.x * nw + w) * nchunks + c) * chunk % span;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(ring + (size_t)s * chunk)), "l"(p), "r"(chunk), "r"(su(&full[s])) : "memory");
      }
    }
  }
  if (acc == 1234.f) sink[0] = acc;
}

// cp.async 16B by all threads: ring of ns chunks of `chunk` bytes, block-wide
__global__ void k_ldgsts(const char* src, int nchunks, int chunk, int ns, size_t span, float* sink) {
  char* ring = (char*)dsm;
  const int tid = threadIdx.x, nt = blockDim.x;
  float acc = 0;
  auto issue = [&](int c) {
    const char* p = src + ((size_t)blockIdx.x * nchunks + c) * chunk % span;
    char* d = ring + (size_t)(c % ns) * chunk;
    for (int o = tid * 16; o < chunk; o += nt * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(d + o)), "l"(p + o) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int c = 0; c < ns - 1 && c < nchunks; ++c) issue(c);
  for (int c = 0; c < nchunks; ++c) {
    if (c + ns - 1 < nchunks) issue(c + ns - 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(3) : "memory");  // ns=4 assumed
    __syncthreads();
    acc += *(float*)(ring + (size_t)(c % ns) * chunk + tid * 4);
    __syncthreads();
  }
  if (acc == 1234.f) sink[0] = acc;
}

int main() {
  size_t span = (size_t)64 << 20;
  char* src; float* sink;
  CK(cudaMalloc(&src, span)); CK(cudaMalloc(&sink, 64)); CK(cudaMemset(src, 0, span));
  CK(cudaFuncSetAttribute(k_bulk_mw, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int nw : {1, 2, 4, 8, 16}) for (int chunk : {1024, 2048, 8192}) for (int ns : {2, 4}) {
    size_t smem = 16 * 8 * 32 + (size_t)nw * ns * chunk;
    if (smem > 200 * 1024) continue;
    int nchunks = (int)((4u << 20) / (nw * chunk));  // 4 MB per CTA
    k_bulk_mw<<<148, nw * 32, smem>>>(src, nchunks, chunk, ns, span, sink);
    cudaEventRecord(a);
    k_bulk_mw<<<148, nw * 32, smem>>>(src, nchunks, chunk, ns, span, sink);
    cudaEventRecord(b); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = 148.0 * nw * nchunks * chunk;
    printf("bulk warps=%2d chunk=%5d ns=%d: per-SM %6.1f GB/s aggregate %6.0f GB/s\n", nw, chunk, ns,
           bytes / 148 / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9);
  }
  for (int nt : {128, 256, 512}) for (int chunk : {8192, 16384}) {
    int ns = 4, nchunks = (int)((4u << 20) / chunk);
    size_t smem = (size_t)ns * chunk;
    k_ldgsts<<<148, nt, smem>>>(src, nchunks, chunk, ns, span, sink);
    cudaEventRecord(a);
    k_ldgsts<<<148, nt, smem>>>(src, nchunks, chunk, ns, span, sink);
    cudaEventRecord(b); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = 148.0 * nchunks * chunk;
    printf("ldgsts threads=%3d chunk=%5d ns=4: per-SM %6.1f GB/s aggregate %6.0f GB/s\n", nt, chunk,
           bytes / 148 / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
