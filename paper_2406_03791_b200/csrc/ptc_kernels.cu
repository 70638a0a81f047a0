// Instantiations of the tensor-core persistent kernel (persistent_tc.cuh).
// A translation unit of their own so ptxas can run at -O1 on them alone: the
// kernel is a latency chain of polls, barriers and short dependent bodies, and
// -O1 scheduling measured 0.6-0.75 us/step faster than -O3 at C2 / C4 (A/B),
// while the throughput kernels in rnntg.cu (encoder projection GEMM, FFMA
// persistent kernel, graph-step kernels) keep -O3.
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/rnntg.h"
#include "common.cuh"
#include "persistent_tc.cuh"

namespace rnntg {

// the tensor-core kernel instantiation for a decode configuration: one per
// (algorithm, cell) for production, the generic one (flags read at run time)
// when the event trace is on
const void* tc_kernel_for(int algo, int cell, bool traced) {
  using namespace ptc;
  if (traced) return (const void*)ptc_kernel<true, SPEC_GENERIC>;
  switch (spec_of(algo, cell)) {
    case spec_of(ALGO_FS, 0): return (const void*)ptc_kernel<false, spec_of(ALGO_FS, 0)>;
    case spec_of(ALGO_FS, 1): return (const void*)ptc_kernel<false, spec_of(ALGO_FS, 1)>;
    case spec_of(ALGO_LL, 0): return (const void*)ptc_kernel<false, spec_of(ALGO_LL, 0)>;
    case spec_of(ALGO_LL, 1): return (const void*)ptc_kernel<false, spec_of(ALGO_LL, 1)>;
    case spec_of(ALGO_TDT, 0): return (const void*)ptc_kernel<false, spec_of(ALGO_TDT, 0)>;
    default: return (const void*)ptc_kernel<false, spec_of(ALGO_TDT, 1)>;
  }
}

}  // namespace rnntg
