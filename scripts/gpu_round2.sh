#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1c}
echo "=== pytest -m gpu"; timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
echo "=== bench c2"; timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; tail -c 400 gpurun_out/bench_c2_${TAG}.json
echo "=== bench c5 (N=1, B=256 T=500)"; timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err; tail -c 400 gpurun_out/bench_c5_${TAG}.json; tail -3 gpurun_out/bench_c5_${TAG}.err
echo "=== torchrun 2 ranks sharing the GPU (functional check of the N>1 path)"
RNNTG_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-compare > gpurun_out/bench_n2share_${TAG}.json 2> gpurun_out/bench_n2share_${TAG}.err; tail -c 400 gpurun_out/bench_n2share_${TAG}.json; tail -3 gpurun_out/bench_n2share_${TAG}.err
echo "=== reference arm"; timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1; tail -c 500 gpurun_out/bench_ref_${TAG}.json
