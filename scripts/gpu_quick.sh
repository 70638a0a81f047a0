#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 240 python scripts/quick_persistent.py 2>&1 | tail -20
echo "rc=$?"
