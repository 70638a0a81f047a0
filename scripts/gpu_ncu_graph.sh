#!/bin/bash
# ncu of the graph step kernels (standalone launches after one decode)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=20 timeout 600 ncu --set full --clock-control none --import-source on \
  -k "regex:pred_layer|pred_proj|joint_kernel" -s 8 -c 6 -o gpurun_out/prof_graph_${TAG:-r1b} -f \
  python scripts/prof_kernels.py > gpurun_out/ncu_graph.log 2>&1
tail -3 gpurun_out/ncu_graph.log
./tests/cpp/test_dropin 2>&1 | tail -12
