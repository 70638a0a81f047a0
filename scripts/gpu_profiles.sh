#!/bin/bash
# Profiles for profiles/: ncu launch list of one bench-like decode and a full
# ncu capture of the dominant kernels; nsys timeline of the graph executor.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
# launch list (per-launch device time) of one persistent decode and one graph decode
T=250 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_persistent_${TAG}.csv python scripts/prof_kernels_exec.py persistent > /dev/null 2>&1
T=40 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_graph_${TAG}.csv python scripts/prof_kernels_exec.py graph > /dev/null 2>&1
# full capture: persistent kernel (1 launch) and K1 (tcgen05) and graph step kernels
T=50 timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:persistent_kernel|encproj_tc" -c 2 -o gpurun_out/prof_persistent_${TAG} -f \
  python scripts/prof_kernels_exec.py persistent > gpurun_out/ncu_persistent_${TAG}.log 2>&1
T=20 timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:pred_layer|pred_proj|joint_kernel" -s 8 -c 4 -o gpurun_out/prof_graph_${TAG} -f \
  python scripts/prof_kernels_exec.py graph > gpurun_out/ncu_graph_${TAG}.log 2>&1
# nsys timeline of a graph decode (kernel intervals -> GPU idle fraction)
NSYS=/opt/nvidia/nsight-compute/2025.2.1/host/target-linux-x64/nsys
if [ -x "$NSYS" ]; then
  T=250 timeout 600 $NSYS profile --cuda-graph-trace=node -t cuda -o gpurun_out/nsys_graph_${TAG} -f true \
    python scripts/prof_kernels_exec.py graph > gpurun_out/nsys_graph_${TAG}.log 2>&1
  timeout 300 $NSYS stats --report cuda_gpu_trace --format csv -o gpurun_out/nsys_graph_${TAG} \
    gpurun_out/nsys_graph_${TAG}.nsys-rep > /dev/null 2>&1
fi
ls -la gpurun_out
