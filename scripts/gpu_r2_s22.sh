#!/bin/bash
# round 2 session 22: K1 prep occupancy variants (warps per CTA, wedge stack size)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s22
timeout 300 python scripts/quick_timing.py 1 3 > $O.base.log 2>&1
for v in prep_w4_s96 prep_w4_s64 prep_w4_s48 prep_w8_s64; do
  DRK_LIB_PATH=vbuild/$v.so timeout 300 python scripts/quick_timing.py 1 3 > $O.$v.log 2>&1
done
