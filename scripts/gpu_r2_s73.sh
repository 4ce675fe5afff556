#!/bin/bash
# round 2 session 73: config-3 launch list (where the 25 ms sort stage goes)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s73
timeout 900 bash scripts/launch_list.sh 3 $O.launches_c3.csv > $O.launches_c3.md 2>&1
