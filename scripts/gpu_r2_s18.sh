#!/bin/bash
# round 2 session 18: config-3 launch list (r2 kernels) + host trace
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s18
DRK_HOST_TRACE=1 timeout 400 python scripts/quick_timing.py 3 > $O.timing.log 2>&1
timeout 900 bash scripts/launch_list.sh 3 $O.launches_c3.csv > $O.launches_c3.md 2>&1
