#!/bin/bash
# round 2 session 74: converged-warp pop-through variants; host trace of config 3 (sort-stage gap)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s74
for v in "" vbuild/thruw3.so vbuild/thruw4.so "" vbuild/thruw3.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-700; else timeout 400 python scripts/quick_timing.py 1 2 3 2>&1 | cut -c1-700; fi
done > $O.variants.log 2>&1
DRK_HOST_TRACE=1 timeout 300 python scripts/quick_timing.py 3 > $O.trace3.log 2>&1
