// microbench.cu — B200 measurements that decide the persistent design:
//   (1) grid-barrier latency for G co-resident CTAs (flat vs cluster-tree)
//   (2) broadcast activation streaming: every CTA bulk-copies the same 8 KB
//       chunks (no multicast) vs distinct chunks vs TMA multicast in clusters
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench scripts/microbench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

namespace cg = cooperative_groups;

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// flat barrier (same as persistent.cuh)
__device__ void bar_flat(unsigned* bar, int G, int sleep_ns) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == (unsigned)G - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) {
        if (sleep_ns) __nanosleep(sleep_ns);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// cluster-tree barrier: hardware cluster barrier, one CTA per cluster on the global counter
__device__ void bar_tree(unsigned* bar, int nclusters) {
  __syncthreads();
  cluster_sync_all();
  if (cluster_rank() == 0 && threadIdx.x == 0) {
    const unsigned gen = ld_acquire(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == (unsigned)nclusters - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) {
      }
    }
    __threadfence();
  }
  cluster_sync_all();
}

__global__ void k_barrier_flat(unsigned* bar, int iters, int sleep_ns, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) bar_flat(bar, gridDim.x, sleep_ns);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void k_barrier_cg(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void k_barrier_tree(unsigned* bar, int iters, int nclusters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) bar_tree(bar, nclusters);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// ---------------- streaming
// Each CTA streams `nchunks` chunks of 8 KB into a ring of NS slots; chunk
// source = src + (shared ? c : blockIdx.x * nchunks + c) * 8 KB.  One warp
// consumes (sums) each chunk.  mc > 1: cluster multicast, rank r issues the
// chunks with c % mc == r to every CTA of the cluster.
template <int NS>
__global__ void k_stream(const float* src, int nchunks, int shared, int mc, float* sink,
                         unsigned long long* out) {
  __shared__ __align__(128) float ring[NS][2048];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int tid = threadIdx.x;
  const unsigned rank = mc > 1 ? cluster_rank() : 0;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[i])), "r"(mc));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (mc > 1) cluster_sync_all();
  unsigned long long t0 = clock64();
  float acc = 0.f;
  if (tid == 32) {  // producer
    for (int c = 0; c < nchunks; ++c) {
      const int slot = c % NS;
      if (c >= NS) {
        asm volatile(
            "{.reg .pred p; W1_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W1_%=;}" ::"r"(
                smem_u32(&empty[slot])),
            "r"(((c / NS) - 1) & 1));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8192;" ::"r"(smem_u32(&full[slot])));
      const float* s = src + (size_t)(shared ? c : blockIdx.x * nchunks + c) * 2048;
      if (mc == 1) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(
                smem_u32(ring[slot])),
            "l"(s), "r"(smem_u32(&full[slot]))
            : "memory");
      } else if ((unsigned)(c % mc) == rank) {
        const unsigned short mask = (unsigned short)((1u << mc) - 1);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], 8192, [%2], %3;" ::"r"(
                smem_u32(ring[slot])),
            "l"(s), "r"(smem_u32(&full[slot])), "h"(mask)
            : "memory");
      }
    }
  } else if (tid < 32) {  // consumer warp
    for (int c = 0; c < nchunks; ++c) {
      const int slot = c % NS;
      asm volatile(
          "{.reg .pred p; W2_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W2_%=;}" ::"r"(
              smem_u32(&full[slot])),
          "r"((c / NS) & 1));
      for (int i = tid; i < 2048; i += 32) acc += ring[slot][i];
      __syncwarp();
      if (tid == 0) {
        if (mc == 1) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])));
        } else {
          for (int r = 0; r < mc; ++r) {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[slot])), "r"(r));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote));
          }
        }
      }
    }
  }
  __syncthreads();
  if (mc > 1) cluster_sync_all();
  if (tid == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
  if (acc == 12345.f) sink[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("SMs %d, clock %d MHz\n", nsm, clk_khz / 1000);
  unsigned* bar;
  unsigned long long* out;
  CK(cudaMalloc(&bar, 64));
  CK(cudaMalloc(&out, 64));
  unsigned long long h;
  const int iters = 2000;
  for (int G : {32, 64, 128, 148}) {
    for (int sleep : {0, 32}) {
      CK(cudaMemset(bar, 0, 64));
      int sl = sleep, it = iters;
      void* args[] = {&bar, &it, &sl, &out};
      CK(cudaLaunchCooperativeKernel((void*)k_barrier_flat, G, 256, args, 0, 0));
      CK(cudaDeviceSynchronize());
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      CK(cudaLaunchCooperativeKernel((void*)k_barrier_flat, G, 256, args, 0, 0));
      cudaEventRecord(b);
      CK(cudaDeviceSynchronize());
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("flat barrier G=%3d sleep=%2d: %.3f us/barrier\n", G, sleep, 1000 * ms / iters);
    }
    {
      int it = iters;
      void* args[] = {&it, &out};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      CK(cudaLaunchCooperativeKernel((void*)k_barrier_cg, G, 256, args, 0, 0));
      cudaEventRecord(a);
      CK(cudaLaunchCooperativeKernel((void*)k_barrier_cg, G, 256, args, 0, 0));
      cudaEventRecord(b);
      CK(cudaDeviceSynchronize());
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("cg grid.sync G=%3d: %.3f us/barrier\n", G, 1000 * ms / iters);
    }
    for (int cs : {2, 4, 8}) {
      if (G % cs) continue;
      CK(cudaMemset(bar, 0, 64));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = G;
      cfg.blockDim = 256;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      int ncl = G / cs, it = iters;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_barrier_tree, bar, it, ncl, out);
      if (e != cudaSuccess) {
        printf("tree barrier G=%d cluster %d: launch failed: %s\n", G, cs, cudaGetErrorString(e));
        cudaGetLastError();
        continue;
      }
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      CK(cudaLaunchKernelEx(&cfg, k_barrier_tree, bar, it, ncl, out));
      cudaEventRecord(b);
      CK(cudaDeviceSynchronize());
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("tree barrier G=%3d cluster=%d: %.3f us/barrier\n", G, cs, 1000 * ms / iters);
    }
  }
  // streaming
  const int nchunks = 400;
  float* src;
  float* sink;
  CK(cudaMalloc(&src, (size_t)nsm * nchunks * 8192));
  CK(cudaMalloc(&sink, nsm * 4));
  CK(cudaMemset(src, 0, (size_t)nsm * nchunks * 8192));
  for (int G : {128, 148}) {
    for (int shared : {1, 0}) {
      for (int mc : {1, 2, 4}) {
        if (G % mc) continue;
        if (!shared && mc > 1) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = G;
        cfg.blockDim = 64;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = mc;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = nchunks, sh = shared, m = mc;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          cudaEventRecord(a);
          CK(cudaLaunchKernelEx(&cfg, k_stream<4>, (const float*)src, nc, sh, m, sink, out));
          cudaEventRecord(b);
          CK(cudaDeviceSynchronize());
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep)
            printf("stream G=%3d %s mc=%d: %.3f us/chunk/CTA, aggregate delivered %.1f GB/s\n", G,
                   shared ? "shared " : "distinct", mc, 1000 * ms / nchunks,
                   (double)G * nchunks * 8192 / (ms * 1e-3) / 1e9);
        }
      }
    }
  }
  return 0;
}
