#!/bin/bash
# ncu capture of the step kernels (standalone launches after one decode).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export T=${T:-20}
timeout 300 python scripts/prof_kernels.py
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:pred_layer|pred_proj|joint_kernel" -s ${SKIP:-0} -c ${COUNT:-4} \
  -o gpurun_out/prof_${TAG:-r1} -f python scripts/prof_kernels.py > gpurun_out/ncu_${TAG:-r1}.log 2>&1
tail -5 gpurun_out/ncu_${TAG:-r1}.log
