// encproj_tc.cuh — K1, the one-shot encoder projection fp = x @ enc_proj over
// all B*T frames (joint.enc_proj of model.cpp:365-369, hoisted out of the
// decode loop), on the 5th-generation tensor cores.
//
// Precision: 3xTF32.  x = x_hi + x_lo with x_hi = x & 0xffffe000 (exact split);
// likewise enc_proj = w_hi + w_lo (split once on the host).  Each 8-deep k
// step issues three tcgen05.mma.kind::tf32 into the same TMEM accumulator:
// x_hi*w_hi + x_hi*w_lo + x_lo*w_hi, giving ~1e-6 relative error (plain TF32
// is ~1e-4, outside the budget: SURVEY.md §7 hard part 1).
//
// Structure (one 128 x BN output tile per CTA, 6 warps):
//   warp 0      TMA producer: x tile [128 m x 32 k] and w_hi / w_lo tiles
//               [BN n x 32 k], SWIZZLE_128B, into a 3-stage ring (mbarriers)
//   warps 2..5  split x in place into x_hi and a second x_lo buffer
//               (elementwise, so the swizzled layout is preserved), then
//               fence.proxy.async and signal the MMA warp
//   warp 1      TMEM allocation + single-thread tcgen05.mma issue; commits
//               free the stage and finally signal the epilogue
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> registers -> global
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "kernels.cuh"

namespace rnntg {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;       // fp32 k per stage = 128 bytes = one swizzle row
constexpr int STAGES = 3;
constexpr int NTHR = 192;
constexpr int TILE_A = BM * BK * 4;  // 16 KB

__host__ __device__ inline size_t smem_bytes(int BN) {
  const size_t stage = 2 * (size_t)TILE_A + 2 * (size_t)BN * BK * 4;
  return 1024 + STAGES * stage + 256;
}

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  // K-major, SWIZZLE_128B canonical layout: 8-row groups 1024 B apart (SBO),
  // LBO unused (1), version 1 (sm100), layout type 2 (128B swizzle).
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(NTHR, 1)
    encproj_tc_kernel(const __grid_constant__ CUtensorMap map_x,
                      const __grid_constant__ CUtensorMap map_whi,
                      const __grid_constant__ CUtensorMap map_wlo, float* __restrict__ out, int M,
                      int Kp, int Jp, int BN) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-aligned stage buffers
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const size_t stage_bytes = 2 * (size_t)TILE_A + 2 * (size_t)BN * BK * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * stage_bytes);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* accb = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accb + 1);
  auto sA = [&](int s) { return base + s * stage_bytes; };
  auto sAlo = [&](int s) { return base + s * stage_bytes + TILE_A; };
  auto sBhi = [&](int s) { return base + s * stage_bytes + 2 * TILE_A; };
  auto sBlo = [&](int s) { return base + s * stage_bytes + 2 * TILE_A + (size_t)BN * BK * 4; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = Kp / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accb, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = TILE_A + 2 * BN * BK * 4;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_load_2d(sA(s), &map_x, kb * BK, m0, &full[s]);
        tma_load_2d(sBhi(s), &map_whi, kb * BK, n0, &full[s]);
        tma_load_2d(sBlo(s), &map_wlo, kb * BK, n0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&conv[s], (kb / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t ahi = sdesc_sw128(smem_u32(sA(s)));
        const uint64_t alo = sdesc_sw128(smem_u32(sAlo(s)));
        const uint64_t bhi = sdesc_sw128(smem_u32(sBhi(s)));
        const uint64_t blo = sdesc_sw128(smem_u32(sBlo(s)));
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint64_t dk = (uint64_t)(k * 32 >> 4);  // +32 bytes per 8 tf32
          mma_tf32(tmem, ahi + dk, bhi + dk, idesc, (kb | k) != 0);
          mma_tf32(tmem, ahi + dk, blo + dk, idesc, 1);
          mma_tf32(tmem, alo + dk, bhi + dk, idesc, 1);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accb);
    }
    __syncwarp();
  } else {
    // converter: x -> (x_hi in place, x_lo), 128 threads x 128 bytes each
    const int ct = threadIdx.x - 64;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      float4* a = reinterpret_cast<float4*>(sA(s));
      float4* lo = reinterpret_cast<float4*>(sAlo(s));
#pragma unroll
      for (int i = 0; i < TILE_A / 16 / 128; ++i) {
        const int o = ct + 128 * i;
        float4 v = a[o], h, l;
        h.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
        h.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
        h.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
        h.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
        l.x = v.x - h.x;
        l.y = v.y - h.y;
        l.z = v.z - h.z;
        l.w = v.w - h.w;
        a[o] = h;
        lo[o] = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&conv[s])) : "memory");
    }
    // epilogue
    mbar_wait(accb, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = m0 + 32 * q + lane;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%"
          "15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
            "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
            "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < M) {
        float4* dst = reinterpret_cast<float4*>(out + (size_t)row * Jp + n0 + c0);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          dst[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                               __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
  }
}

}  // namespace tc

// ------------------------------------------------------------------ host
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode_tiled() {
  static PFN_encodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

inline bool make_map_2d(CUtensorMap* map, const float* ptr, uint64_t inner, uint64_t outer,
                        uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled enc = get_encode_tiled();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner * sizeof(float)};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Projection plan for one (x, out, rows) triple: tensor maps are built once.
struct EncPlan {
  CUtensorMap mx, mhi, mlo;
  int M = 0, Kp = 0, Jp = 0, BN = 0;
  const float* x = nullptr;
  float* out = nullptr;
  bool ok = false;
};

inline bool encproj_tc_supported(const DevModel& M) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) return false;
  if (!get_encode_tiled()) return false;
  if (M.Fp % tc::BK != 0 || M.Jp % 64 != 0) return false;
  // the attribute is per function, shared by every model: set the largest tile's need
  return cudaFuncSetAttribute(tc::encproj_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)tc::smem_bytes(128)) == cudaSuccess;
}

// x: [rows][Fp] (pitched, zero-padded), out: [rows][Jp].
inline bool encproj_plan(EncPlan& p, const DevModel& M, const float* x, float* out, int rows) {
  p.M = rows;
  p.Kp = M.Fp;
  p.Jp = M.Jp;
  p.BN = M.Jp % 128 == 0 ? 128 : 64;
  p.x = x;
  p.out = out;
  p.ok = make_map_2d(&p.mx, x, (uint64_t)M.Fp, (uint64_t)rows, tc::BK, tc::BM) &&
         make_map_2d(&p.mhi, M.enc_hi, (uint64_t)M.Fp, (uint64_t)M.Jp, tc::BK, (uint32_t)p.BN) &&
         make_map_2d(&p.mlo, M.enc_lo, (uint64_t)M.Fp, (uint64_t)M.Jp, tc::BK, (uint32_t)p.BN);
  return p.ok;
}

inline dim3 encproj_grid(const EncPlan& p) { return dim3(p.Jp / p.BN, (p.M + tc::BM - 1) / tc::BM); }

inline cudaError_t encproj_launch(const EncPlan& p, cudaStream_t s) {
  tc::encproj_tc_kernel<<<encproj_grid(p), tc::NTHR, tc::smem_bytes(p.BN), s>>>(
      p.mx, p.mhi, p.mlo, p.out, p.M, p.Kp, p.Jp, p.BN);
  return cudaGetLastError();
}

// Graph node for the projection (kernel params copied into the node).
inline cudaError_t encproj_add_node(cudaGraph_t g, cudaGraphNode_t* last, bool* last_kernel,
                                    EncPlan& p) {
  void* args[8] = {&p.mx, &p.mhi, &p.mlo, &p.out, &p.M, &p.Kp, &p.Jp, &p.BN};
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeKernel;
  np.kernel.func = (void*)tc::encproj_tc_kernel;
  np.kernel.gridDim = encproj_grid(p);
  np.kernel.blockDim = dim3(tc::NTHR);
  np.kernel.sharedMemBytes = (unsigned)tc::smem_bytes(p.BN);
  np.kernel.kernelParams = args;
  cudaGraphNode_t n;
  cudaError_t e = cudaGraphAddNode(&n, g, *last ? last : nullptr, *last ? 1 : 0, &np);
  if (e != cudaSuccess) return e;
  *last = n;
  *last_kernel = true;
  return cudaSuccess;
}

}  // namespace rnntg
