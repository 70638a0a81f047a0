#!/bin/bash
# quick correctness + trace of the tensor-core executor
cd "${GRAFT_REPO_ROOT:-/root/repo}"
NSEEDS=${NSEEDS:-3} timeout 300 python scripts/quick_tc.py 2>&1 | grep -v "^\s*$" | cut -c1-220 | tail -14
timeout 200 python scripts/trace_tc.py 2>&1 | tail -17
