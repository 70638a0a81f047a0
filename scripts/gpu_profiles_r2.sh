#!/bin/bash
# Round-2 bench profiles: every BASELINE config on the default executor (with
# the other executors and the CPU reference in alt_exec / cpu_baseline), the
# realistic-emission regime (blank bias 0.015), the graph executor line, C5.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # name args...
  local n=$1; shift
  timeout 900 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/r2_bench_$n.json 2> gpurun_out/r2_bench_$n.err
  echo "$n rc=$?"; tail -2 gpurun_out/r2_bench_$n.err
}
run c2
run c2_graph --exec graph --no-cpu-baseline
run c2_bias --blank-bias 0.015
run c3 --config c3 --no-cpu-baseline
run c3_bias --config c3 --blank-bias 0.015 --no-cpu-baseline --steps 60
run c4 --config c4 --no-cpu-baseline --steps 60
run c1 --config c1 --no-cpu-baseline --steps 40
run c5_n1 --config c5 --no-cpu-baseline
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference_arm.json 2>&1; echo "ref rc=$?"
