#!/bin/bash
# round 2 session 78: early bracket lookup in the backward (atan2 form) vs off
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s78
for v in "" vbuild/bwd_noebr.so "" vbuild/bwd_noebr.so; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 400 python scripts/quick_timing.py 2 2>&1 | cut -c1-420; else timeout 400 python scripts/quick_timing.py 2 2>&1 | cut -c1-420; fi
done > $O.variants.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_det.py -m gpu -q -x > $O.parity.log 2>&1
echo "rc=$?" >> $O.parity.log
