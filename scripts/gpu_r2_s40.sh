#!/bin/bash
# round 2 session 40: reference-precision forward, warp per pixel vs thread per pixel
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s40
timeout 300 python scripts/fp64_all_probe.py > $O.log 2>&1
DRK_FP64_ALL=thread timeout 300 python scripts/fp64_all_probe.py >> $O.log 2>&1
