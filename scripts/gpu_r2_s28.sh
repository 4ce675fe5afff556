#!/bin/bash
# round 2 session 28: radix sort items per thread (8 / 12 / 16)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s28
for v in base rs12 rs16; do
  if [ $v = base ]; then L=""; else L=vbuild/$v.so; fi
  DRK_LIB_PATH=$L timeout 400 python scripts/quick_timing.py 1 3 > $O.$v.log 2>&1
  DRK_LIB_PATH=$L timeout 600 python scripts/config4_probe.py 2 > $O.$v.c4.log 2>&1
done
