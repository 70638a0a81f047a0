#!/bin/bash
# Round-2 ncu evidence: the launch list of the default bench command, a full
# capture of K6 (C2, tensor executor), of one graph step launch (graph
# executor) and of K1, summarised into profiles/ by scripts/ncu_summary.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-compare --no-cpu-baseline \
  > gpurun_out/r2_launches_c2.log 2>&1; echo "launches rc=$?"
RNNTG_LAUNCH_GRAPH=0 T=250 timeout 900 ncu --set full --import-source on --clock-control none -k regex:ptc_kernel -c 1 \
  -o gpurun_out/r2_ncu_tc -f python scripts/prof_kernels_exec.py tensor > gpurun_out/r2_ncu_tc.log 2>&1; echo "tc rc=$?"
# the graph executor's body kernel (step launches), launched by the host loop
# (ncu does not profile kernels in conditional-node bodies)
T=20 timeout 900 ncu --set full --import-source on --clock-control none -k regex:ptc_kernel -s 30 -c 1 \
  -o gpurun_out/r2_ncu_step -f python scripts/prof_kernels_exec.py hostloop > gpurun_out/r2_ncu_step.log 2>&1; echo "step rc=$?"
T=250 timeout 900 ncu --set full --import-source on --clock-control none -k regex:encproj -c 1 \
  -o gpurun_out/r2_ncu_k1 -f python scripts/prof_kernels_exec.py tensor > gpurun_out/r2_ncu_k1.log 2>&1; echo "k1 rc=$?"
ls -la gpurun_out/*.ncu-rep
