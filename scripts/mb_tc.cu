// mb_tc.cu — microbenchmarks that fix the design of the tensor-core
// persistent decoder (persistent_tc.cuh):
//   1. correctness of kind::f16 MMAs with A from shared memory (SS) and A
//      from tensor memory (TS), fp16 hi/lo split, swap-AB (M = 128 weight
//      rows, N = batch rows), checked against a double-precision host dot;
//   2. cycles per 16-deep k step for the MMA mixes the decoder can use
//      (W_hi SS N=64 + W_lo TS/SS N=32, ...), 1 CTA and 148 CTAs;
//   3. cross-CTA hop latency: 8 KB written by 128 threads + release counter
//      -> acquire poll -> bulk copy into shared memory (ping-pong).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_tc scripts/mb_tc.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

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
__device__ __forceinline__ uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// issued by a whole (converged) warp; elect.sync picks the issuing lane
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
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su(bar)) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void minit(uint64_t* bar, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// byte offset of (row r, k) inside a [rows x 64] fp16 K-major SWIZZLE_128B tile
__host__ __device__ inline uint32_t swz(int r, int k) {
  return (uint32_t)(r * 128 + ((((k * 2) >> 4) ^ (r & 7)) << 4) + ((k * 2) & 15));
}

// ---------------------------------------------------------------- test 1/2
// smem: Whi [KC][128 x 64] fp16 (16 KB per chunk), Wlo same, B [KC][64 x 64] (8 KB)
// mode 0: correctness (KC chunks, out[128][96] = D1 | D2)
// mode 1..: timing loops over the same chunks `reps` times
//   1: SS(Whi,N=64) + TS(Wlo,N=32)   2: SS(Whi,N=64) + SS(Wlo,N=32)
//   3: TS(Whi,N=64) + TS(Wlo,N=32)   4: SS(Whi,N=64) only  5: TS N=32 only  6: SS N=96 single
template <int mode>
__global__ void __launch_bounds__(128, 1) k_mma(const __half* whi, const __half* wlo, const __half* bm, int KC,
                                                int reps, float* out, long long* cyc) {
  unsigned char* sWhi = dsm;
  unsigned char* sWlo = dsm + KC * 16384;
  unsigned char* sB = dsm + 2 * KC * 16384;
  uint64_t* bar = (uint64_t*)(sB + KC * 32768);
  uint32_t* tslot = (uint32_t*)(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // load tiles (already swizzled on host)
  for (int i = tid; i < KC * 16384 / 16; i += 128) {
    ((int4*)sWhi)[i] = ((const int4*)whi)[i];
    ((int4*)sWlo)[i] = ((const int4*)wlo)[i];
  }
  for (int i = tid; i < KC * 32768 / 16; i += 128) ((int4*)sB)[i] = ((const int4*)bm)[i];
  if (tid == 0) {
    minit(&bar[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  // W_lo (and W_hi for mode 3) into TMEM: row = lane, column c = k pair (2c, 2c+1)
  // TMEM columns: [0,96) accumulators, [128, 128+32*KC) Wlo, [256, 256+32*KC) Whi
  {
    const int row = 32 * warp + lane;
    for (int kc = 0; kc < KC; ++kc)
      for (int c8 = 0; c8 < 4; ++c8) {  // 8 columns = 16 k per store
        uint32_t rl[8], rh[8];
        for (int j = 0; j < 8; ++j) {
          const int k = c8 * 16 + 2 * j;
          const uint32_t lo0 = *(const uint16_t*)(sWlo + kc * 16384 + swz(row, k));
          const uint32_t lo1 = *(const uint16_t*)(sWlo + kc * 16384 + swz(row, k + 1));
          const uint32_t hi0 = *(const uint16_t*)(sWhi + kc * 16384 + swz(row, k));
          const uint32_t hi1 = *(const uint16_t*)(sWhi + kc * 16384 + swz(row, k + 1));
          rl[j] = lo0 | (lo1 << 16);
          rh[j] = hi0 | (hi1 << 16);
        }
        const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
        tmem_st8(tmem + lane_off + 256 + kc * 32 + c8 * 8, rl);
        if (KC <= 4) tmem_st8(tmem + lane_off + 384 + kc * 32 + c8 * 8, rh);
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint32_t i64 = idesc_f16(128, 64), i32 = idesc_f16(128, 32), i128 = idesc_f16(128, 128),
                   i256 = idesc_f16(128, 256);
    const uint32_t d1 = tmem, d2 = tmem + 64;
    long long t0 = clock64();
    const int R = mode == 0 ? 1 : reps;
    for (int rep = 0; rep < R; ++rep)
      for (int kc = 0; kc < KC; ++kc) {
        const uint64_t ah = sdesc(su(sWhi + kc * 16384)), al = sdesc(su(sWlo + kc * 16384));
        const uint64_t b = sdesc(su(sB + kc * 32768));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t acc = (rep | kc | k) != 0;
          const uint64_t dk = (uint64_t)(k * 32 >> 4);
          const uint32_t tl = tmem + 256 + kc * 32 + k * 8, th = tmem + 384 + kc * 32 + k * 8;
          switch (mode) {
            case 0: [[fallthrough]];
            case 1: mma_ss(d1, ah + dk, b + dk, i64, acc); mma_ts(d2, tl, b + dk, i32, acc); break;
            case 2: mma_ss(d1, ah + dk, b + dk, i64, acc); mma_ss(d2, al + dk, b + dk, i32, acc); break;
            case 3: mma_ts(d1, th, b + dk, i64, acc); mma_ts(d2, tl, b + dk, i32, acc); break;
            case 4: mma_ss(d1, ah + dk, b + dk, i64, acc); break;
            case 5: mma_ts(d2, tl, b + dk, i32, acc); break;
            case 6: mma_ss(d1, ah + dk, b + dk, i256, acc); break;
            case 7: mma_ss(tmem + 64 * (k & 3), ah + dk, b + dk, i64, (rep | kc) != 0); break;
            case 8: mma_ss(d1, ah + dk, b + dk, i128, acc); break;
            case 9: mma_ss(d1, ah + dk, b + dk, i32, acc); break;
            case 10:
              mma_ss(tmem + 96 * (k & 1), ah + dk, b + dk, i64, (rep | kc | (k >> 1)) != 0);
              mma_ts(tmem + 96 * (k & 1) + 64, tl, b + dk, i32, (rep | kc | (k >> 1)) != 0);
              break;
            case 11: mma_ts(tmem + 32 * (k & 3), tl, b + dk, i32, (rep | kc) != 0); break;
          }
        }
      }
    __syncwarp();
    long long ti = clock64();
    commit(&bar[0]);
    mwait(&bar[0], 0);
    long long t1 = clock64();
    if (cyc && lane == 0) {
      cyc[blockIdx.x] = t1 - t0;
      cyc[256 + blockIdx.x] = ti - t0;
    }
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (mode == 0 && blockIdx.x == 0) {
    const int row = 32 * warp + lane;
    float v[32];
    for (int c = 0; c < 96; c += 32) {
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
      for (int i = 0; i < 32; ++i) out[row * 96 + c + i] = v[i];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---------------------------------------------------------------- test 3
// CTA 0 and CTA 1 (different SMs) ping-pong a [64 x 64] fp16 chunk (8 KB):
// writer: 128 threads st.global 64 B each, bar.sync, thread 0 publishes
// (variant 0: fence.proxy.async.global + red.release.gpu; variant 1: __threadfence + atomicAdd)
// reader: lane 0 polls ld.acquire.gpu, then cp.async.bulk 8 KB -> smem, mbarrier wait.
__global__ void __launch_bounds__(128, 1) k_hop(unsigned char* buf0, unsigned char* buf1, unsigned* ctr, int iters,
                                                int variant, long long* out) {
  unsigned char* s = dsm;
  uint64_t* bar = (uint64_t*)(dsm + 8192);
  const int tid = threadIdx.x, me = blockIdx.x;
  if (me > 1) return;
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
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const bool my_turn_first = me == 0;
    for (int half = 0; half < 2; ++half) {
      const bool write = (half == 0) == my_turn_first;
      if (write) {
        int4 v = make_int4(it, tid, half, me);
        int4* d = (int4*)mine;
        for (int i = tid; i < 512; i += 128) d[i] = v;
        if (variant == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
          if (variant == 0)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(myc) : "memory");
          else {
            __threadfence();
            atomicAdd(myc, 1u);
          }
        }
      } else {
        if (tid == 0) {
          unsigned cur;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(thc) : "memory");
          } while (cur < (unsigned)(it + 1));
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(8192) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(s)),
                       "l"(theirs), "r"(8192), "r"(su(bar))
                       : "memory");
          mwait(bar, ph);
        }
        ph ^= 1;
        __syncthreads();
      }
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[me] = t1 - t0;
}

// ---------------------------------------------------------------- host
static uint16_t h16(float f) { __half h = __float2half_rn(f); return *(uint16_t*)&h; }
static float f16(uint16_t u) { __half h; *(uint16_t*)&h = u; return __half2float(h); }

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d clock %d MHz\n", nsm, clk / 1000);
  const int KC = 2;  // 128 k
  const int K = KC * 64;
  // W [128 x K] scaled by 2^7, A [32 x K]
  std::vector<float> W(128 * K), A(32 * K);
  srand(1);
  for (auto& w : W) w = ((rand() / (float)RAND_MAX) * 0.16f - 0.08f);
  for (auto& a : A) a = ((rand() / (float)RAND_MAX) * 2.f - 1.f);
  const float ws = 128.f;
  std::vector<uint16_t> hWhi(KC * 128 * 64), hWlo(KC * 128 * 64), hB(KC * 256 * 64);
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < K; ++k) {
      const float w = W[r * K + k] * ws;
      const uint16_t hi = h16(w);
      const uint16_t lo = h16(w - f16(hi));
      const int kc = k / 64, kk = k % 64;
      hWhi[kc * 8192 + swz(r, kk) / 2] = hi;
      hWlo[kc * 8192 + swz(r, kk) / 2] = lo;
    }
  for (int r = 0; r < 32; ++r)
    for (int k = 0; k < K; ++k) {
      const float a = A[r * K + k];
      const uint16_t hi = h16(a), lo = h16(a - f16(hi));
      const int kc = k / 64, kk = k % 64;
      hB[kc * 16384 + swz(r, kk) / 2] = hi;
      hB[kc * 16384 + swz(32 + r, kk) / 2] = lo;
    }
  __half *dWhi, *dWlo, *dB;
  float* dout;
  long long* dcyc;
  CK(cudaMalloc(&dWhi, hWhi.size() * 2));
  CK(cudaMalloc(&dWlo, hWlo.size() * 2));
  CK(cudaMalloc(&dB, hB.size() * 2));
  CK(cudaMalloc(&dout, 128 * 96 * 4));
  CK(cudaMalloc(&dcyc, 512 * 8));
  CK(cudaMemcpy(dWhi, hWhi.data(), hWhi.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dWlo, hWlo.data(), hWlo.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  const size_t smem = 2 * KC * 16384 + KC * 32768 + 64;
#define SETA(m) CK(cudaFuncSetAttribute(k_mma<m>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SETA(0) SETA(1) SETA(2) SETA(3) SETA(4) SETA(5) SETA(6) SETA(7) SETA(8) SETA(9) SETA(10) SETA(11)
  k_mma<0><<<1, 128, smem>>>(dWhi, dWlo, dB, KC, 1, dout, dcyc);
  CK(cudaDeviceSynchronize());
  std::vector<float> out(128 * 96);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  double maxrel = 0, maxrel_hi_only = 0;
  for (int r = 0; r < 128; ++r)
    for (int b = 0; b < 32; ++b) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)W[r * K + k] * (double)A[b * K + k];
      const double got = ((double)out[r * 96 + b] + ((double)out[r * 96 + 32 + b] + (double)out[r * 96 + 64 + b])) / ws;
      const double hi_only = (double)out[r * 96 + b] / ws;
      const double den = 0.05;  // ~ rms of the dots
      maxrel = fmax(maxrel, fabs(got - ref) / den);
      maxrel_hi_only = fmax(maxrel_hi_only, fabs(hi_only - ref) / den);
    }
  printf("correctness SS(Whi)+TS(Wlo) fp16 hi/lo: max rel err %.3e (hi*hi only %.3e)\n", maxrel, maxrel_hi_only);
  // timing
  const char* names[] = {"", "SS Whi N64 + TS Wlo N32", "SS Whi N64 + SS Wlo N32", "TS Whi N64 + TS Wlo N32",
                         "SS Whi N64 only", "TS Wlo N32 only", "SS N256 1 acc",
                         "SS N64 4 rotating acc", "SS N128 1 acc", "SS N32 1 acc", "SS64+TS32 2 rotating pairs",
                         "TS N32 4 rotating acc"};
  const int reps = 200;
  for (int mode = 1; mode <= 11; ++mode) {
    for (int grid : {1, nsm}) {
      auto run = [&](int r) {
        switch (mode) {
#define RUNM(m) case m: k_mma<m><<<grid, 128, smem>>>(dWhi, dWlo, dB, KC, r, dout, dcyc); break;
          RUNM(1) RUNM(2) RUNM(3) RUNM(4) RUNM(5) RUNM(6) RUNM(7) RUNM(8) RUNM(9) RUNM(10) RUNM(11)
        }
      };
      run(10);
      run(reps);
      CK(cudaDeviceSynchronize());
      std::vector<long long> cyc(512);
      CK(cudaMemcpy(cyc.data(), dcyc, 512 * 8, cudaMemcpyDeviceToHost));
      long long mx = 0, mi = 0;
      for (int g = 0; g < grid; ++g) { mx = cyc[g] > mx ? cyc[g] : mx; mi = cyc[256 + g] > mi ? cyc[256 + g] : mi; }
      printf("mode %d %-26s grid %3d: %.1f cycles per 16-k step (issue %.1f)\n", mode, names[mode], grid,
             (double)mx / (reps * KC * 4), (double)mi / (reps * KC * 4));
    }
  }
  // hop latency
  unsigned char *b0, *b1;
  unsigned* ctr;
  long long* dh;
  CK(cudaMalloc(&b0, 8192));
  CK(cudaMalloc(&b1, 8192));
  CK(cudaMalloc(&ctr, 256 * 4));
  CK(cudaMalloc(&dh, 16));
  CK(cudaFuncSetAttribute(k_hop, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 + 64));
  for (int variant = 0; variant < 2; ++variant)
    for (int grid : {2, 74, 148}) {
      const int iters = 2000;
      CK(cudaMemset(ctr, 0, 256 * 4));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_hop<<<grid, 128, 8192 + 64>>>(b0, b1, ctr, iters, variant, dh);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h[2];
      CK(cudaMemcpy(h, dh, 16, cudaMemcpyDeviceToHost));
      printf("hop variant %d (grid %d): %.1f cycles / %.3f us per one-way hop (8 KB + counter)\n", variant, grid,
             (double)h[0] / (2 * iters), 1000.0 * ms / (2 * iters));
    }
  return 0;
}
