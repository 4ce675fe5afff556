#!/bin/bash
# round 2 session 54: forward raster at 3 CTAs / SM (80 registers, no TMA staging) vs 2
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s54
for v in base tma0 fast768; do
  if [ $v = base ]; then L=""; else L=vbuild/$v.so; fi
  DRK_LIB_PATH=$L timeout 300 python scripts/quick_timing.py 1 2 > $O.$v.log 2>&1
done
