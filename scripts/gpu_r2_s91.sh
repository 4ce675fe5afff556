#!/bin/bash
# round 2 session 91: whole-tile pop-through fast path and TMA staging off, re-measured after the batch change
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s91
for v in "" vbuild/thru1.so vbuild/notma.so "" vbuild/thru1.so vbuild/notma.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 2>&1 | cut -c1-300; else timeout 400 python scripts/quick_timing.py 1 2 2>&1 | cut -c1-300; fi
done > $O.variants.log 2>&1
