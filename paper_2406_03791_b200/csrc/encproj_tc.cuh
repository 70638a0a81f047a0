// encproj_tc.cuh — K1, the one-shot encoder projection fp = x @ enc_proj over
// all B*T frames (joint.enc_proj of model.cpp:365-369, hoisted out of the
// decode loop).  Launch helpers shared by the decode graph and the C ABI.
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace rnntg {

inline bool encproj_tc_supported(const DevModel&) { return false; }

inline cudaError_t launch_encproj(const DevModel& M, bool /*tc*/, const float* x, float* out,
                                  int rows, cudaStream_t s) {
  encproj_simt_kernel<<<dim3(M.Jp / 64, (rows + 63) / 64), 256, 0, s>>>(x, M.enc, out, rows, M.F,
                                                                       M.Jp);
  return cudaGetLastError();
}

inline cudaError_t encproj_add_node(cudaGraph_t g, cudaGraphNode_t* last, bool* last_kernel,
                                    const DevModel& M, bool /*tc*/, const float* x, float* out,
                                    int rows) {
  const float* enc = M.enc;
  int Mr = rows, F = M.F, Jp = M.Jp;
  void* args[6] = {&x, &enc, &out, &Mr, &F, &Jp};
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeKernel;
  p.kernel.func = (void*)encproj_simt_kernel;
  p.kernel.gridDim = dim3(M.Jp / 64, (rows + 63) / 64);
  p.kernel.blockDim = dim3(256);
  p.kernel.sharedMemBytes = 0;
  p.kernel.kernelParams = args;
  cudaGraphNode_t n;
  cudaError_t e = cudaGraphAddNode(&n, g, *last ? last : nullptr, *last ? 1 : 0, &p);
  if (e != cudaSuccess) return e;
  *last = n;
  *last_kernel = true;
  return cudaSuccess;
}

}  // namespace rnntg
