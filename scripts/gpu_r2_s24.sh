#!/bin/bash
# round 2 session 24: config-4 forward+backward launch list (r2 kernels) and stage probe
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s24
timeout 900 python scripts/config4_probe.py 2 bwd > $O.c4probe.log 2>&1
timeout 1500 bash scripts/launch_list.sh 4 $O.launches_c4.csv bwd > $O.launches_c4.md 2>&1
