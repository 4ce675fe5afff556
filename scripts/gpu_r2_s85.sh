#!/bin/bash
# round 2 session 85: batch size sweep (whole-tile 128 default vs 64; half-tile 128 vs 64)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s85
for v in "" vbuild/b64.so vbuild/h64.so "" vbuild/b64.so vbuild/h64.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-300; else timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-300; fi
done > $O.variants.log 2>&1
