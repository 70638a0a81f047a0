#!/bin/bash
# End-of-session check: smoke, every GPU test, the bench lines (C2 with the CPU
# baseline, C1/C3/C4/C5, N=2 sharing the GPU, the reference arm), the tensor
# launch list and one ncu --set full capture of the persistent kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1n}
echo "=== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
echo "=== pytest -m gpu"; timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
echo "=== bench c2"; timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; tail -2 gpurun_out/bench_c2_${TAG}.err
for c in c1 c3 c4; do echo "=== bench $c"; timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err; tail -1 gpurun_out/bench_${c}_${TAG}.err; done
echo "=== bench c5 N=1"; timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-compare > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err; tail -1 gpurun_out/bench_c5_${TAG}.err
echo "=== torchrun 2 ranks sharing the GPU"
RNNTG_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-compare > gpurun_out/bench_n2share_${TAG}.json 2> gpurun_out/bench_n2share_${TAG}.err; tail -1 gpurun_out/bench_n2share_${TAG}.err
echo "=== reference arm"; timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; tail -c 300 gpurun_out/bench_ref_${TAG}.json
echo "=== ncu"; TAG=$TAG bash scripts/gpu_profiles_tc.sh
python - <<PY
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_*_${TAG}.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f.split("/")[-1], d.get("config", {}).get("exec"), round(d.get("value", 0)), d.get("unit"), "us/step", d.get("us_per_step"), "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
PY
