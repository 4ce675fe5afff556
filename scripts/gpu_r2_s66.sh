#!/bin/bash
# round 2 session 66: backward with record_grad_fast out of line
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s66
for i in 1 2; do
timeout 300 python scripts/quick_timing.py 2 > $O.base_$i.log 2>&1
DRK_LIB_PATH=vbuild/rgf_noinl.so timeout 300 python scripts/quick_timing.py 2 > $O.noinl_$i.log 2>&1
done
