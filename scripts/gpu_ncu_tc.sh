#!/bin/bash
# ncu capture of the tensor-core persistent kernel (source-level stall sampling)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-tc}
T=${T:-100} timeout 900 ncu --set full --import-source on --clock-control none -k regex:ptc_kernel -c 1 \
  -o gpurun_out/ncu_${TAG} -f python scripts/prof_kernels_exec.py tensor > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
ls -la gpurun_out/ncu_${TAG}.ncu-rep
