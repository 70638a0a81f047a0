#!/bin/bash
# ncu launch list of one bench-like decode (tensor executor) + full capture of ptc_kernel and K1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1tc}
T=250 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_tensor_${TAG}.csv python scripts/prof_kernels_exec.py tensor > /dev/null 2>&1
T=250 timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:ptc_kernel|encproj_tc" -c 2 -o gpurun_out/ncu_tc_${TAG} -f \
  python scripts/prof_kernels_exec.py tensor > gpurun_out/ncu_tc_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_tc_${TAG}.log
ls -la gpurun_out | grep ${TAG}
