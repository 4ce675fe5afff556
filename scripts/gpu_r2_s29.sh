#!/bin/bash
# round 2 session 29: cost of the per-pixel backward state on forward-only frames
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s29
for i in 1 2; do
timeout 300 python scripts/e2e_probe.py 1 >> $O.log 2>&1
DRK_NO_STATE=1 timeout 300 python scripts/e2e_probe.py 1 >> $O.log 2>&1
done
timeout 300 python scripts/quick_timing.py 1 >> $O.log 2>&1
DRK_NO_STATE=1 timeout 300 python scripts/quick_timing.py 1 >> $O.log 2>&1
