#!/bin/bash
# round 2 session 75: device-time trace of the binning sort phases (configs 1 and 3)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s75
DRK_SORT_TRACE=1 timeout 300 python scripts/quick_timing.py 1 3 > $O.sorttrace.log 2>&1
