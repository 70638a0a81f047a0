#!/bin/bash
# GPU tests + C2 bench (tensor executor default) + C3/C4 lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1e}
echo "=== pytest -m gpu"; timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
echo "=== bench c2"; timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; tail -c 300 gpurun_out/bench_c2_${TAG}.json; tail -2 gpurun_out/bench_c2_${TAG}.err
for c in c3 c4; do echo "=== bench $c"; timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err; tail -c 200 gpurun_out/bench_${c}_${TAG}.json; tail -2 gpurun_out/bench_${c}_${TAG}.err; done
