// mb_mma.cu — tensor-pipe rate of the tensor executor's MMA shapes, operands
// resident (no copies): cycles per 16-deep k-step over 40 k-steps (one
// 128-row tile, K = 640), from the first issue to the commit's mbarrier.
//   c0  TS N=64 + SS N=32   (W_hi in TMEM, W_lo in smem: the executor today)
//   c1  SS N=64 + TS N=32   (W_hi in smem, W_lo in TMEM)
//   c2  TS N=64 only        c3  SS N=32 only
//   c4  SS N=64 only        c5  TS N=32 only
//   c6  TS N=96 only        c7  SS N=96 only
//   c8  TS N=64 + TS N=32   (both A operands in TMEM)
//   c9  SS N=64 + SS N=32   (both in smem)
//   c10 TS N=64 M=64        c11 SS N=32 M=64     c12 TS N=64 + SS N=32, M=64
//   c13 SS N=64 + SS N=32, M=64
//   c14 TS N=64 + TS N=32 into the SAME accumulator columns 0..31
//   c15 TS N=64 + SS N=32 into the same columns
//   c16 executor layout, LO_TMEM: D cols 0..63, W_hi A at 64 + 8 ks, W_lo A at 384 + 8 ks
//       for ks < 16 (TS + TS), SS W_lo for ks >= 16, all into D
//   c17 executor layout before: D1 0..63, D2 64..95, W_hi A at 192 + 8 ks (TS), SS W_lo into D2
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_mma scripts/mb_mma.cu
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
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su(bar))
      : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
          su(bar)),
      "r"(ph)
      : "memory");
}

constexpr int KSTEPS = 40;
template <int C>
__global__ void __launch_bounds__(128, 1) k_mma(long long* out, int reps) {
  // smem: A (W) [10 chunks][16 KB] at 0, B ring [4][8 KB] at 160 KB, barrier after
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm + 160 * 1024 + 48 * 1024);  // ring + N=96 overrun room
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    const uint32_t a0 = su(dsm), b0 = su(dsm + 160 * 1024);
    const uint32_t d1 = tmem, d2 = tmem + 96, ta = tmem + 192;  // A in TMEM from column 192
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      const long long t0 = clock64();
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) {
        const int kc = ks >> 2, k = ks & 3, st = kc & 3;
        const uint64_t ad = sdesc(a0 + kc * 16384) + 2 * k, bd = sdesc(b0 + st * 8192) + 2 * k;
        const uint32_t at = ta + (ks * 8) % 320;
        const uint32_t acc = ks != 0;
        if (C == 0) { mma_ts(d1, at, bd, idesc_f16(128, 64), acc); mma_ss(d2, ad, bd, idesc_f16(128, 32), acc); }
        if (C == 1) { mma_ss(d1, ad, bd, idesc_f16(128, 64), acc); mma_ts(d2, at, bd, idesc_f16(128, 32), acc); }
        if (C == 2) mma_ts(d1, at, bd, idesc_f16(128, 64), acc);
        if (C == 3) mma_ss(d2, ad, bd, idesc_f16(128, 32), acc);
        if (C == 4) mma_ss(d1, ad, bd, idesc_f16(128, 64), acc);
        if (C == 5) mma_ts(d2, at, bd, idesc_f16(128, 32), acc);
        if (C == 6) mma_ts(d1, at, bd, idesc_f16(128, 96), acc);
        if (C == 7) mma_ss(d1, ad, bd, idesc_f16(128, 96), acc);
        if (C == 8) { mma_ts(d1, at, bd, idesc_f16(128, 64), acc); mma_ts(d2, at, bd, idesc_f16(128, 32), acc); }
        if (C == 9) { mma_ss(d1, ad, bd, idesc_f16(128, 64), acc); mma_ss(d2, ad, bd, idesc_f16(128, 32), acc); }
        if (C == 10) mma_ts(d1, at, bd, idesc_f16(64, 64), acc);
        if (C == 11) mma_ss(d2, ad, bd, idesc_f16(64, 32), acc);
        if (C == 12) { mma_ts(d1, at, bd, idesc_f16(64, 64), acc); mma_ss(d2, ad, bd, idesc_f16(64, 32), acc); }
        if (C == 16) {
          mma_ts(tmem, tmem + 64 + ks * 8, bd, idesc_f16(128, 64), acc);
          if (ks < 16) mma_ts(tmem, tmem + 384 + ks * 8, bd, idesc_f16(128, 32), 1);
          else mma_ss(tmem, ad, bd, idesc_f16(128, 32), 1);
        }
        if (C == 17) {
          mma_ts(tmem, tmem + 192 + ks * 8, bd, idesc_f16(128, 64), acc);
          mma_ss(tmem + 64, ad, bd, idesc_f16(128, 32), acc);
        }
        if (C == 14) { mma_ts(d1, at, bd, idesc_f16(128, 64), acc); mma_ts(d1, at, bd, idesc_f16(128, 32), 1); }
        if (C == 15) { mma_ts(d1, at, bd, idesc_f16(128, 64), acc); mma_ss(d1, ad, bd, idesc_f16(128, 32), 1); }
        if (C == 13) { mma_ss(d1, ad, bd, idesc_f16(64, 64), acc); mma_ss(d2, ad, bd, idesc_f16(64, 32), acc); }
      }
      commit(bar);
      mwait(bar, r & 1);
      const long long t1 = clock64();
      if (r > 0) tot += t1 - t0;
    }
    if (threadIdx.x == 0) out[C] = tot / (reps - 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int C>
void run(const char* name, long long* dout) {
  const int smem = 160 * 1024 + 48 * 1024 + 64;
  CK(cudaFuncSetAttribute(k_mma<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_mma<C><<<1, 128, smem>>>(dout, 20);
  CK(cudaDeviceSynchronize());
  long long h[32];
  CK(cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost));
  printf("%-26s %6lld cycles / 40 k-steps = %5.1f per k-step\n", name, h[C], h[C] / 40.0);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  long long* dout;
  CK(cudaMalloc(&dout, 32 * 8));
  CK(cudaMemset(dout, 0, 32 * 8));
  run<0>("c0 TS64 + SS32 (today)", dout);
  run<1>("c1 SS64 + TS32", dout);
  run<2>("c2 TS64", dout);
  run<3>("c3 SS32", dout);
  run<4>("c4 SS64", dout);
  run<5>("c5 TS32", dout);
  run<16>("c16 executor LO_TMEM layout", dout);
  run<17>("c17 executor previous layout", dout);
  run<14>("c14 TS64 + TS32 same D", dout);
  run<15>("c15 TS64 + SS32 same D", dout);
  run<6>("c6 TS96", dout);
  run<7>("c7 SS96", dout);
  run<9>("c9 SS64 + SS32", dout);
  run<11>("c11 SS32 M64", dout);
  run<13>("c13 SS64 + SS32 M64", dout);
  run<10>("c10 TS64 M64", dout);
  run<12>("c12 TS64 + SS32 M64", dout);
  run<8>("c8 TS64 + TS32", dout);
  return 0;
}
