#!/bin/bash
# round 2 session 51: radix scatter ranks by match.any instead of 9 ballots
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s51
for v in base rs_match rs_match16; do
  if [ $v = base ]; then L=""; else L=vbuild/$v.so; fi
  DRK_LIB_PATH=$L timeout 300 python scripts/quick_timing.py 1 3 > $O.$v.log 2>&1
done
DRK_LIB_PATH=vbuild/rs_match.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > $O.tests.log 2>&1
