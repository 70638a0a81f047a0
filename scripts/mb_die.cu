// mb_die.cu — is a cross-CTA hand-off slower across the two B200 dies?
// 148 CTAs (one per SM) record their %smid; CTA 0 ping-pongs a relaxed 8-byte
// word with CTA k (k = 1..147, one pair at a time, the rest idle); the
// one-way latency per pair is printed with both SM ids.  A bimodal
// distribution separates same-die from cross-die pairs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/mb_die scripts/mb_die.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void k_pair(unsigned long long* a, unsigned long long* b, int partner, int iters, int* smid,
                       long long* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) smid[blockIdx.x] = (int)s;
  const int me = blockIdx.x;
  if (me != 0 && me != partner) return;
  if (threadIdx.x != 0) return;
  const bool ping = me == 0;
  const long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    if (ping) {
      str(a, (unsigned long long)it);
      while (ldr(b) != (unsigned long long)it) {
      }
    } else {
      while (ldr(a) != (unsigned long long)it) {
      }
      str(b, (unsigned long long)it);
    }
  }
  const long long t1 = clock64();
  if (ping) out[partner] = (t1 - t0) / (2 * iters);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *a, *b;
  int* smid;
  long long* out;
  CK(cudaMalloc(&a, 256));
  CK(cudaMalloc(&b, 256));
  CK(cudaMalloc(&smid, nsm * 4));
  CK(cudaMalloc(&out, nsm * 8));
  CK(cudaMemset(out, 0, nsm * 8));
  for (int k = 1; k < nsm; ++k) {
    CK(cudaMemset(a, 0, 256));
    CK(cudaMemset(b, 0, 256));
    k_pair<<<nsm, 32>>>(a, b, k, 500, smid, out);
    CK(cudaDeviceSynchronize());
  }
  std::vector<long long> h(nsm);
  std::vector<int> sm(nsm);
  CK(cudaMemcpy(h.data(), out, nsm * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(sm.data(), smid, nsm * 4, cudaMemcpyDeviceToHost));
  printf("CTA0 on SM %d\n", sm[0]);
  std::vector<long long> v(h.begin() + 1, h.end());
  std::sort(v.begin(), v.end());
  printf("one-way hop cycles: min %lld p25 %lld median %lld p75 %lld max %lld\n", v[0], v[v.size() / 4],
         v[v.size() / 2], v[3 * v.size() / 4], v.back());
  for (int k = 1; k < nsm; ++k) printf("cta %3d sm %3d : %lld\n", k, sm[k], h[k]);
  return 0;
}
