// mb_pipe2.cu — the tensor executor's load + MMA round under kernel-like
// conditions, to find what slows the tensor pipe inside the executor (91
// cycles per 16-deep k-step there vs 63 with operands resident, mb_mma.cu).
// One CTA of 10 warps: warp 0 = converged producer (2-D TMA, 8 KB chunks, 4-stage
// ring reset every round), warp 1 = MMA issuer, warps 2-9 = "epilogue" waiting
// on the accumulator barrier in a try_wait loop.  Cycles per round of 10 chunks (40 k-steps), chunk-0 issue -> acc.
//   L0  D1 [0,64) D2 [64,96): TS W_hi (TMEM @192) N=64 -> D1, SS W_lo N=32 -> D2
//   L1  D [0,64): TS W_hi (TMEM @64) N=64, W_lo TS (TMEM @384) chunks 0-3 / SS after, into D[0,32)
//   L2  D [0,64): TS W_hi (TMEM @128) N=64, SS W_lo into D[0,32) (same columns)
//   L3  as L0 without the ring: chunks resident, no TMA (MMA only)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_pipe2 scripts/mb_pipe2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>
#include <cuda_fp16.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

constexpr int KC = 10, NST = 4, CH = 8192;
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
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
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
__device__ __forceinline__ void arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(bar)) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(p));
  return p != 0;
}

static __device__ __constant__ int RANDW_DUMMY = 0;
#define RANDW (SPIN == 2)
template <int L, int SPIN>
__global__ void __launch_bounds__(320, 1) k_pipe2(const __grid_constant__ CUtensorMap map, int rounds, long long* out) {
  unsigned char* wsm = dsm;                    // [KC][16 KB] W_lo smem image
  unsigned char* ring = dsm + KC * 16384;      // [NST][8 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + NST * CH);
  uint64_t *full = bars, *empty = bars + NST, *accf = bars + 2 * NST, *cmd = accf + 1, *acce = cmd + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acce + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(accf)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(cmd)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su(acce)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (RANDW) {  // random fp16 weights in smem (W_lo image) and TMEM (W_hi columns)
    uint32_t st = 777u + threadIdx.x * 7919u;
    uint32_t* w = reinterpret_cast<uint32_t*>(wsm);
    for (int i = threadIdx.x; i < KC * 16384 / 4; i += blockDim.x) {
      st = st * 1664525u + 1013904223u;
      w[i] = (st & 0x3bff3bffu);  // two fp16 in (-1, 1)
    }
    if (warp >= 2 && warp < 6) {
      const int q = warp & 3;
      for (int c = 64; c < 512; c += 8) {
        uint32_t r[8];
        for (int j = 0; j < 8; ++j) {
          st = st * 1664525u + 1013904223u;
          r[j] = st & 0x3bff3bffu;
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         tmem + ((uint32_t)(32 * q) << 16) + c),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  constexpr uint32_t ID64 = idesc(128, 64), ID32 = idesc(128, 32);
  if (warp == 0) {
    uint32_t eb = 0;
    for (int r = 0; r < rounds; ++r) {
      mwait(cmd, r & 1);
      if (L == 3) continue;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int st = kc % NST;
        if (kc >= NST) mwait(&empty[st], ((eb >> st) & 1u) ^ 1u);
        eb ^= 1u << st;
        if (elect_one()) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(CH) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  su(ring + st * CH)),
              "l"(&map), "r"(64 * kc), "r"(64 * (r & 1)), "r"(su(&full[st]))
              : "memory");
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    uint32_t fb = 0;
    const uint32_t w0 = su(wsm), rg = su(ring);
    long long tot = 0;
    for (int r = 0; r < rounds; ++r) {
      if (r >= 1) mwait(acce, (r - 1) & 1);
      const long long t0 = clock64();
      if (elect_one()) arrive(cmd);
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int st = kc % NST;
        if (L != 3) {
          mwait(&full[st], (fb >> st) & 1u);
          fb ^= 1u << st;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        const uint64_t ad = sdesc(w0 + kc * 16384), bd = sdesc(rg + st * CH);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t acc = (kc | k) != 0;
          if (L == 0 || L == 3) {
            mma_ts(tmem, tmem + 192 + kc * 32 + k * 8, bd + 2 * k, ID64, acc);
            mma_ss(tmem + 64, ad + 2 * k, bd + 2 * k, ID32, acc);
          } else if (L == 1) {
            mma_ts(tmem, tmem + 64 + kc * 32 + k * 8, bd + 2 * k, ID64, acc);
            if (kc < 4) mma_ts(tmem, tmem + 384 + kc * 32 + k * 8, bd + 2 * k, ID32, 1);
            else mma_ss(tmem, ad + 2 * k, bd + 2 * k, ID32, 1);
          } else {
            mma_ts(tmem, tmem + 128 + kc * 32 + k * 8, bd + 2 * k, ID64, acc);
            mma_ss(tmem, ad + 2 * k, bd + 2 * k, ID32, 1);
          }
        }
        if (L != 3) commit(&empty[st]);
      }
      commit(accf);
      mwait(accf, r & 1);
      const long long t1 = clock64();
      if (r >= 2) tot += t1 - t0;
    }
    if (lane == 0 && blockIdx.x == 0) out[L * 3 + SPIN] = tot / (rounds - 2);
  } else {
    for (int r = 0; r < rounds; ++r) {
      mwait(accf, r & 1);  // (SPIN is always 1: the executor's epilogue spins)
      if (lane == 0) arrive(acce);
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int L, int SPIN>
void run(const char* name, const CUtensorMap& map, long long* dout, int grid = 1) {
  const int smem = KC * 16384 + NST * CH + 256;
  CK(cudaFuncSetAttribute(k_pipe2<L, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_pipe2<L, SPIN><<<grid, 320, smem>>>(map, 200, dout);  // every CTA streams the same activations
  CK(cudaDeviceSynchronize());
  long long h[32];
  CK(cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost));
  printf("%-56s %6lld cycles / round = %5.1f per k-step\n", name, h[L * 3 + SPIN], h[L * 3 + SPIN] / 40.0);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned char* act;
  long long* dout;
  CK(cudaMalloc(&act, 128 * 640 * 2));
  if (getenv("ZERO_ACT")) {
    CK(cudaMemset(act, 0, 128 * 640 * 2));
  } else {  // random fp16 activations in (-1, 1)
    std::vector<uint16_t> h(128 * 640);
    uint32_t st = 12345;
    for (auto& v : h) {
      st = st * 1664525u + 1013904223u;
      const float f = ((st >> 8) / 16777216.0f) * 2.0f - 1.0f;
      __half hv = __float2half(f);
      memcpy(&v, &hv, 2);
    }
    CK(cudaMemcpy(act, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&dout, 32 * 8));
  CK(cudaMemset(dout, 0, 32 * 8));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap map;
  const cuuint64_t dims[2] = {640, 128};
  const cuuint64_t strides[1] = {640 * 2};
  const cuuint32_t box[2] = {64, 64};
  const cuuint32_t es[2] = {1, 1};
  if (((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, act, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  run<3, 1>("L3 resident operands (no ring), epilogue spinning", map, dout);
  run<0, 1>("L0 executor before (TS->D1, SS->D2), epilogue spinning", map, dout);
  run<1, 1>("L1 LO_TMEM layout, epilogue spinning", map, dout);
  run<2, 1>("L2 same-column SS lo, epilogue spinning", map, dout);
  run<0, 2>("L0 random weights + activations", map, dout);
  run<1, 2>("L1 random weights + activations", map, dout);
  run<3, 2>("L3 random weights (resident)", map, dout);
  return 0;
}
