#!/bin/bash
# round 2 session 59: pop-through fast path in the fast backward
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s59
for i in 1 2; do
timeout 300 python scripts/quick_timing.py 2 > $O.base_$i.log 2>&1
DRK_LIB_PATH=vbuild/bwd_thru.so timeout 300 python scripts/quick_timing.py 2 > $O.thru_$i.log 2>&1
done
