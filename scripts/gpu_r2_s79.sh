#!/bin/bash
# round 2 session 79: L1 prefetch of the SH coefficients past the bracket bound (forward)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s79
for v in "" vbuild/shpf.so "" vbuild/shpf.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-300; else timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-300; fi
done > $O.variants.log 2>&1
