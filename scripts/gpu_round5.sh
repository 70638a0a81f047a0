#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1h}
for c in c1 c3 c4; do echo "=== bench $c"; timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err; tail -2 gpurun_out/bench_${c}_${TAG}.err; done
echo "=== bench c5 N=1"; timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-compare > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err; tail -2 gpurun_out/bench_c5_${TAG}.err
echo "=== torchrun 2 ranks sharing the GPU"
RNNTG_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-compare > gpurun_out/bench_n2share_${TAG}.json 2> gpurun_out/bench_n2share_${TAG}.err; tail -2 gpurun_out/bench_n2share_${TAG}.err
python - <<PY
import json, glob
for f in sorted(glob.glob("gpurun_out/*_${TAG}.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f.split("/")[-1], d["config"].get("exec"), round(d["value"]), "frames/s", round(d.get("us_per_step", 0), 2), "us/step", "n_gpus", d["n_gpus"])
    for a in d.get("alt_exec") or []: print("   alt", a.get("exec"), a.get("us_per_step"), a.get("value"), a.get("unavailable"))
PY
