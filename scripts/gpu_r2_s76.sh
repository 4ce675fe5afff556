#!/bin/bash
# round 2 session 76: bracket loads ahead of the radius reject; loop-top barrier removed
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s76
for v in "" vbuild/ebr.so vbuild/notop.so vbuild/ebr_notop.so "" vbuild/ebr.so vbuild/ebr_notop.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-300; else timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-300; fi
done > $O.variants.log 2>&1
