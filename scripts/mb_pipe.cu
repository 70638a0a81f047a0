// mb_pipe.cu — the tensor-core executor's producer/MMA pipeline in isolation:
// W_hi [KC x 16 KB] resident in smem, W_lo in TMEM, activation chunks (8 KB)
// streamed by 1-D bulk copies into a ring, SS(N=64) + TS(N=32) MMAs per
// 16-k step, per-chunk commits to the ring's empty barriers.  Variants:
//   v0  as in persistent_tc.cuh (tcgen05.fence after every full wait)
//   v1  no tcgen05.fence::after_thread_sync after the full waits
//   v2  chunks already resident (no copies): MMA issue rate only
//   v3  v0 with 2-stage ring
//   v4  v0 with 8 k-steps unrolled across two chunks (commit every 2 chunks)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_pipe scripts/mb_pipe.cu
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
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) { return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24); }
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su(bar))
               : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void minit(uint64_t* bar, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(n) : "memory");
}

constexpr int KC = 10, CHUNK = 8192;

template <int V, int NST>
__global__ void __launch_bounds__(128, 1) k_pipe(const unsigned char* act, int rounds, long long* out) {
  unsigned char* whi = dsm;
  unsigned char* ring = dsm + KC * 16384;
  uint64_t* full = (uint64_t*)(ring + NST * CHUNK);
  uint64_t* empty = full + 8;
  uint64_t* accb = empty + 8;
  uint32_t* tslot = (uint32_t*)(accb + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      minit(&full[i], 1);
      minit(&empty[i], 1);
    }
    minit(&accb[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    if (V != 2 && V != 5 && V != 6) {
      long long issued = 0;
      for (int r = 0; r < rounds; ++r)
        for (int kc = 0; kc < KC; ++kc) {
          const int s = (int)(issued % NST);
          if (issued >= NST) mwait(&empty[s], (uint32_t)(((issued / NST) - 1) & 1));
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(CHUNK) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           su(ring + s * CHUNK)),
                       "l"(act + (size_t)kc * CHUNK), "r"(CHUNK), "r"(su(&full[s]))
                       : "memory");
          ++issued;
        }
    }
  } else if (warp == 1) {
    constexpr uint32_t ID64 = idesc_f16(128, 64), ID32 = idesc_f16(128, 32);
    const uint32_t whi0 = su(whi), ring0 = su(ring);
    long long used = 0;
    if (V == 5 || V == 6) {
      // resident chunks: pure issue-rate test; V5 = 2 MMAs per k step, V6 = SS N64 only
      const long long w0 = clock64();
      for (int r = 0; r < rounds; ++r) {
        const uint32_t d1 = tmem + (r & 1) * 96, d2 = d1 + 64;
        for (int kc = 0; kc < KC; ++kc) {
          const uint64_t ad = sdesc(whi0 + kc * 16384), bd = sdesc(ring0 + (kc & 3) * CHUNK);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            mma_ss(d1, ad + 2 * k, bd + 2 * k, ID64, 1);
            if (V == 5) mma_ts(d2, tmem + 192 + kc * 32 + k * 8, bd + 2 * k, ID32, 1);
          }
        }
      }
      commit(&accb[0]);
      mwait(&accb[0], 0);
      const long long w1 = clock64();
      if (lane == 0) out[blockIdx.x] = w1 - w0;
    } else
    for (int r = 0; r < rounds; ++r) {
      const uint32_t d1 = tmem + (r & 1) * 96, d2 = d1 + 64;
      for (int kc = 0; kc < KC; ++kc) {
        const int s = (int)(used % NST);
        if (V != 2) {
          mwait(&full[s], (uint32_t)((used / NST) & 1));
          if (V != 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        const uint64_t ad = sdesc(whi0 + kc * 16384), bd = sdesc(ring0 + s * CHUNK);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t acc = (kc | k) != 0;
          mma_ss(d1, ad + 2 * k, bd + 2 * k, ID64, acc);
          mma_ts(d2, tmem + 192 + kc * 32 + k * 8, bd + 2 * k, ID32, acc);
        }
        if (V != 2) commit(&empty[s]);
        ++used;
      }
    }
    if (V != 5 && V != 6) {
      commit(&accb[0]);
      mwait(&accb[0], 0);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && V != 5 && V != 6) out[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int V, int NST>
void run(const char* name, const unsigned char* act, long long* dout, int grid) {
  const size_t smem = KC * 16384 + NST * CHUNK + 256;
  CK(cudaFuncSetAttribute(k_pipe<V, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int rounds = 200;
  k_pipe<V, NST><<<grid, 128, smem>>>(act, 4, dout);
  k_pipe<V, NST><<<grid, 128, smem>>>(act, rounds, dout);
  CK(cudaDeviceSynchronize());
  long long h[148];
  CK(cudaMemcpy(h, dout, grid * 8, cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-44s grid %3d: %.0f cycles per 10-chunk round (%.1f per 16-k step)\n", name, grid, (double)mx / rounds,
         (double)mx / rounds / 40);
}

int main() {
  unsigned char* act;
  long long* dout;
  CK(cudaMalloc(&act, KC * CHUNK));
  CK(cudaMemset(act, 0, KC * CHUNK));
  CK(cudaMalloc(&dout, 148 * 8));
  for (int grid : {1, 74}) {
    run<0, 4>("v0 kernel loop (fence after full wait)", act, dout, grid);
    run<1, 4>("v1 no tcgen05 fence", act, dout, grid);
    run<5, 4>("v5 resident, 2 MMAs/k, no waits", act, dout, grid);
    run<6, 4>("v6 resident, SS N64 only", act, dout, grid);
    run<0, 2>("v3 2-stage ring", act, dout, grid);
    run<0, 6>("v0 6-stage ring", act, dout, grid);
  }
  return 0;
}
