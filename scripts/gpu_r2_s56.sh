#!/bin/bash
# round 2 session 56: pop-through fast path with one pop_eval call site (per lane / warp-uniform)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s56
for v in base thru1 thru2; do
  if [ $v = base ]; then L=""; else L=vbuild/$v.so; fi
  DRK_LIB_PATH=$L timeout 300 python scripts/quick_timing.py 1 2 3 > $O.$v.log 2>&1
done
