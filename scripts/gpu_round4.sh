#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1f}
echo "=== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -7
echo "=== pytest -m gpu"; timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
echo "=== bench c2"; timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; tail -2 gpurun_out/bench_c2_${TAG}.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c2_${TAG}.json").read().strip().splitlines()[-1])
print(d["config"]["exec"], round(d["value"]), round(d["us_per_step"],2), "idle", d.get("gpu_idle_pct"), "e2e", round(d["e2e"]["value"]))
for a in d["alt_exec"] or []: print("  alt", a.get("exec"), a.get("us_per_step"), a.get("value"), (a.get("gpu_idle") or {}).get("idle_pct"), a.get("unavailable"))
PY
