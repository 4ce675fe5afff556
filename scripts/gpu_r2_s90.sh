#!/bin/bash
# round 2 session 90: half-tile forward batch 64 (product) vs 32
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s90
for v in "" vbuild/h32.so "" vbuild/h32.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 2 3 2>&1 | cut -c1-300; else timeout 400 python scripts/quick_timing.py 2 3 2>&1 | cut -c1-300; fi
done > $O.variants.log 2>&1
DRK_LIB_PATH=vbuild/h32.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > $O.parity_h32.log 2>&1
echo "rc=$?" >> $O.parity_h32.log
