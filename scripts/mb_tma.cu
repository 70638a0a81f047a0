// mb_tma.cu — issue-to-issue cost of back-to-back 2-D TMA loads from one
// thread (the tensor executor's ring producer issues 10 x 8 KB boxes per round
// and measured ~335 cycles between issues).
//   t0  map in a __grid_constant__ kernel parameter
//   t1  t0 + prefetch.tensormap once at kernel start
//   t2  map copied to global memory (128-B aligned), passed by pointer
//   t3  t2 + prefetch.tensormap
//   t4  as t0 with an mbarrier try_wait on a completed phase before each issue
//   t5  plain cp.async.bulk 8 KB copies (no tensor map)
// Each issue targets a distinct 8 KB smem slot and mbarrier; the loop stamps
// clock64 before every issue, then waits for all data.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_tma scripts/mb_tma.cu -lcuda
#include <cuda.h>
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

constexpr int NCH = 10, CHUNK = 8192;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
extern __shared__ __align__(1024) unsigned char dsm[];

template <int V>
__global__ void k_tma(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, const unsigned char* src,
                      int reps, long long* out) {
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + NCH * CHUNK);
  uint64_t* done = bars + NCH;
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NCH; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[i])));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(done)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(done)));  // phase 0 complete
  const CUtensorMap* mp = (V == 2 || V == 3) ? gmap : &map;
  if (V == 1 || V == 3) asm volatile("prefetch.tensormap [%0];" ::"l"(mp) : "memory");
  long long acc[NCH];
  for (int i = 0; i < NCH; ++i) acc[i] = 0;
  for (int r = 0; r < reps; ++r) {
    long long t[NCH + 1];
    for (int i = 0; i < NCH; ++i) {
      if (V == 4) {
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                su(done))
            : "memory");
      }
      t[i] = clock64();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[i])), "r"(CHUNK) : "memory");
      if (V == 5) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su(dsm + i * CHUNK)),
                     "l"(src + (size_t)i * CHUNK), "r"(CHUNK), "r"(su(&bars[i]))
                     : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su(dsm + i * CHUNK)),
            "l"(mp), "r"(64 * i), "r"(0), "r"(su(&bars[i]))
            : "memory");
      }
    }
    t[NCH] = clock64();
    for (int i = 0; i < NCH; ++i)
      asm volatile(
          "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
              su(&bars[i])),
          "r"(r & 1)
          : "memory");
    const long long te = clock64();
    if (r > 0) {
      for (int i = 0; i < NCH; ++i) acc[i] += t[i + 1] - t[i];
      out[NCH] += te - t[0];
    }
  }
  for (int i = 0; i < NCH; ++i) out[i] = acc[i] / (reps - 1);
  out[NCH] /= (reps - 1);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int V>
void run(const char* name, const CUtensorMap& map, const CUtensorMap* gmap, const unsigned char* src, long long* dout) {
  const int smem = NCH * CHUNK + 256;
  CK(cudaFuncSetAttribute(k_tma<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaMemset(dout, 0, 64 * 8));
  k_tma<V><<<1, 32, smem>>>(map, gmap, src, 50, dout);
  CK(cudaDeviceSynchronize());
  long long h[NCH + 1];
  CK(cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost));
  printf("%-44s issue gaps:", name);
  for (int i = 0; i < NCH; ++i) printf(" %4lld", h[i]);
  printf("   first issue -> all landed %lld\n", h[NCH]);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned char* src;
  long long* dout;
  CUtensorMap* gmap;
  CK(cudaMalloc(&src, 2 << 20));
  CK(cudaMemset(src, 1, 2 << 20));
  CK(cudaMalloc(&dout, 64 * 8));
  CK(cudaMalloc(&gmap, sizeof(CUtensorMap)));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap map;
  // [128 rows][640] fp16, box 64 x 64, 128-B swizzle (the executor's load map)
  const cuuint64_t dims[2] = {640, 128};
  const cuuint64_t strides[1] = {640 * 2};
  const cuuint32_t box[2] = {64, 64};
  const cuuint32_t es[2] = {1, 1};
  CUresult cr = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)cr);
    return 1;
  }
  CK(cudaMemcpy(gmap, &map, sizeof(map), cudaMemcpyHostToDevice));
  run<0>("t0 param map", map, gmap, src, dout);
  run<1>("t1 param map + prefetch.tensormap", map, gmap, src, dout);
  run<2>("t2 global map", map, gmap, src, dout);
  run<3>("t3 global map + prefetch.tensormap", map, gmap, src, dout);
  run<4>("t4 param map + try_wait (complete) per issue", map, gmap, src, dout);
  run<5>("t5 cp.async.bulk 8 KB", map, gmap, src, dout);
  return 0;
}
