#!/bin/bash
# round 2 session 58: config-4 views with / without the pop-through fast path
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s58
timeout 500 python scripts/config4_probe.py 3 > $O.c4.log 2>&1
DRK_LIB_PATH=vbuild/thru_off.so timeout 500 python scripts/config4_probe.py 3 > $O.c4_off.log 2>&1
