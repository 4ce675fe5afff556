#!/bin/bash
# round 2 session 72: warp-uniform pop-through (forward whole-tile / both kernels, backward), early sharpen-constant loads
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s72
for v in "" vbuild/thruw1.so vbuild/thruw2.so vbuild/early2.so vbuild/bthru2.so "" vbuild/thruw1.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-400; else timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-400; fi
done > $O.variants.log 2>&1
