#!/bin/bash
# Full round check: GPU tests, bench (default + c3/c4 lines), ncu of the persistent kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
echo "=== pytest -m gpu"; timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6
echo "=== bench c2"; timeout 900 python bench.py --steps ${STEPS:-10} --warmup ${WARMUP:-5} > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; tail -c 600 gpurun_out/bench_c2_${TAG}.json
for c in ${EXTRA:-c3 c4}; do
  echo "=== bench $c"; timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err; tail -c 300 gpurun_out/bench_${c}_${TAG}.json
done
if [ -n "$NCU" ]; then
  T=50 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:persistent_kernel" -c 1 \
    -o gpurun_out/prof_persistent_${TAG} -f python scripts/prof_kernels_exec.py persistent > gpurun_out/ncu_persistent_${TAG}.log 2>&1
  tail -2 gpurun_out/ncu_persistent_${TAG}.log
fi
