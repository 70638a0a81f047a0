// mb_dsmem.cu — cost of handing an fp32 partial tile to the other CTA of a
// 2-CTA cluster (split-K reduction for the tensor executor).  256 threads per
// CTA each own 16 floats (as after a TMEM load); one hand-off = every thread's
// 16 floats land in the partner's smem and the partner's mbarrier completes.
// Ping-pong between the two CTAs; one-way cycles = round trip / 2.
//   d0  st.shared::cluster.v4.f32 x4 + mbarrier.arrive.release.cluster (remote), 16 KB
//   d1  st.async...mbarrier::complete_tx::bytes.v4.b32 x4 (expect_tx by receiver), 16 KB
//   d2  local STS.128 x4 + fence.proxy.async + bar + 1 thread cp.async.bulk
//       smem -> partner smem (complete_tx), 16 KB
//   d3  d1 with 8 KB (threads 0..127 only)
//   d4  d2 with 8 KB
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_dsmem scripts/mb_dsmem.cu
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
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mwait(uint32_t bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(bar),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int V>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) k_ds(int iters, long long* out) {
  __shared__ __align__(128) float4 rx[256 * 4];  // 16 KB receive
  __shared__ __align__(128) float4 tx[256 * 4];  // 16 KB staging (d2/d4)
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x;
  const bool half = V == 3 || V == 4;
  const int nthr = half ? 128 : 256;
  const uint32_t bytes = nthr * 64;
  const uint32_t peer = rank ^ 1;
  if (tid == 0) {
    // d0: 256 remote arrivals complete a phase; d1-d4: one local arrive + tx bytes
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(V == 0 ? 256 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cluster_sync();
  const uint32_t rbar = mapa(su(&bar), peer), rrx = mapa(su(rx), peer);
  float4 v[4];
  for (int j = 0; j < 4; ++j) v[j] = make_float4(tid, j, rank, 1.0f);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const bool send = (it & 1) == (int)rank;  // rank 0 sends on even, rank 1 on odd iterations
    const uint32_t ph = (it >> 1) & 1;
    if (send) {
      if (V == 0) {
        for (int j = 0; j < 4; ++j)
          asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rrx + (tid * 4 + j) * 16),
                       "f"(v[j].x), "f"(v[j].y), "f"(v[j].z), "f"(v[j].w)
                       : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
      } else if (V == 1 || V == 3) {
        if (tid < nthr)
          for (int j = 0; j < 4; ++j)
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                    rrx + (tid * 4 + j) * 16),
                "r"(__float_as_uint(v[j].x)), "r"(__float_as_uint(v[j].y)), "r"(__float_as_uint(v[j].z)),
                "r"(__float_as_uint(v[j].w)), "r"(rbar)
                : "memory");
      } else {
        if (tid < nthr)
          for (int j = 0; j < 4; ++j) tx[tid * 4 + j] = v[j];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rrx),
              "r"(su(tx)), "r"(bytes), "r"(rbar)
              : "memory");
      }
    } else {
      if (V != 0 && tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
      mwait(su(&bar), ph);
      for (int j = 0; j < 4; ++j) v[j] = rx[tid * 4 + j];  // consume
    }
    if (V >= 2) __syncthreads();  // staging buffer reuse (bulk source read is async)
  }
  const long long t1 = clock64();
  if (tid == 0 && rank == 0) out[V] = (t1 - t0) / iters;
  if (tid == 0 && rank == 0) out[8 + V] = (long long)v[0].x;
  cluster_sync();
}

template <int V>
void run(const char* name, long long* dout) {
  k_ds<V><<<2, 256>>>(1000, dout);
  CK(cudaDeviceSynchronize());
  long long h[16];
  CK(cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost));
  printf("%-62s one-way %5lld cycles\n", name, h[V]);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  long long* dout;
  CK(cudaMalloc(&dout, 16 * 8));
  run<0>("d0 st.shared::cluster.v4 + remote arrive.release.cluster, 16 KB", dout);
  run<1>("d1 st.async complete_tx, 16 KB", dout);
  run<2>("d2 STS + bulk smem->dsmem copy, 16 KB", dout);
  run<3>("d3 st.async complete_tx, 8 KB", dout);
  run<4>("d4 STS + bulk smem->dsmem copy, 8 KB", dout);
  return 0;
}
