#!/bin/bash
# One GPU round trip: smoke, GPU parity tests, a short bench.  Run under gpurun.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
echo "=== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
echo "=== pytest -m gpu"; timeout 1200 python -m pytest tests -m gpu -x -q -s ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -40
echo "=== bench"; timeout 900 python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} --cpu-seconds 5 2>&1 | tail -5
